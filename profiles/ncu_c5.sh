#!/usr/bin/env bash
# Full ncu captures of the dominant kernels of one config (pass 0, iterations
# 1-2 unless noted), from the repo root on the GPU box:
#   gpurun --timeout 2400 -- 'bash profiles/ncu_c5.sh r02 c5'
# Keeps the raw/details pages as CSV (gpurun_out/ comes back only under 64 MiB);
# the .ncu-rep of the first capture is kept.
set -u
tag=${1:-r02}
cfg=${2:-c5}
shift 2 || true
mkdir -p gpurun_out
cap() {  # name regex skip count
  local o="gpurun_out/${tag}_${cfg}_$1"
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:$2" --launch-skip "$3" -c "$4" -o "$o" -f python profiles/prof_run.py "$cfg" 1 > "$o.log" 2>&1
  ncu -i "$o.ncu-rep" --page raw --csv > "$o.raw.csv" 2>/dev/null
  ncu -i "$o.ncu-rep" --page details --csv > "$o.details.csv" 2>/dev/null
  if [ "${KEEP_REP:-0}" != 1 ]; then rm -f "$o.ncu-rep"; fi
}
if [ $# -gt 0 ]; then
  cap "$1" "$2" "${3:-1}" "${4:-1}"
else
  cap lm_block '^lvn::.*lm_block' 1 2
  cap hub_chunks 'lm_hub_chunks' 1 2
  cap hub_decide 'lm_hub_decide' 1 1
  cap psort4 'lm_psort<32, 4' 1 1
  cap psort2 'lm_psort<32, 2' 1 1
  cap ag_big_arcs 'ag_big_arcs' 0 2
fi
ls -la gpurun_out
echo done
