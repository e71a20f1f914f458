#!/usr/bin/env bash
# Full ncu captures of single kernels of one config, summarised on the box
# (raw counters + source-line page as CSV; the .ncu-rep is dropped unless
# KEEP_REP=1, so gpurun_out/ stays under the 64 MiB copy-back limit):
#   bash profiles/ncu_kernels.sh <tag> <config> <skip> <regex> [<regex> ...]
set -u
tag=$1; cfg=$2; skip=$3; shift 3
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for k in "$@"; do
  n=$(echo "$k" | tr -dc "a-zA-Z0-9_")
  o="gpurun_out/${tag}_${cfg}_${n}"
  LVN_POOL_NOCACHE=1 timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
    -k "regex:$k" --launch-skip "$skip" --launch-count 1 -o "$o" -f python profiles/prof_run.py "$cfg" 1 > "$o.log" 2>&1
  ncu -i "$o.ncu-rep" --page raw --csv > "$o.raw.csv" 2>/dev/null
  ncu -i "$o.ncu-rep" --page source --csv --print-source cuda,sass > "$o.src.csv" 2>/dev/null
  python profiles/srcprof.py "$o.src.csv" 40 > "$o.src.txt" 2>&1
  rm -f "$o.src.csv"
  if [ "${KEEP_REP:-0}" != 1 ]; then rm -f "$o.ncu-rep"; fi
done
ls -la gpurun_out
