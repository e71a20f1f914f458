#!/usr/bin/env bash
# Round profile collection (run on the GPU box under gpurun from the repo root):
#   gpurun --timeout 2400 -- 'bash profiles/collect.sh c5'
# Writes raw captures to gpurun_out/ (CSV only: the copy-back limit is 64 MiB);
# profiles/summarize.py turns them into the committed summaries under profiles/.
set -u
cfg=${1:-c5}
export PYTHONPATH=$PWD:$PWD/tests
mkdir -p gpurun_out
# 1. the bench line itself (no profiler attached)
timeout 1200 python bench.py --config "$cfg" > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
# 2. launch list of the same command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$cfg.csv \
  python bench.py --config "$cfg" --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# 3. dram traffic of every local-moving launch of one Louvain run
LVN_POOL_NOCACHE=1 timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:'^lm_' --csv --log-file gpurun_out/move_traffic_$cfg.csv \
  python profiles/prof_run.py "$cfg" 1 > gpurun_out/move_traffic_$cfg.log 2>&1
# 4. full capture of the dominant sort-bin kernel (pass 0, second sweep), raw page only
LVN_POOL_NOCACHE=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:lm_psort<.int.16, .int.4' --launch-skip 16 --launch-count 1 -o gpurun_out/prof_lm_sort_$cfg -f \
  python profiles/prof_run.py "$cfg" 1 > gpurun_out/prof_lm_sort_$cfg.log 2>&1
ncu -i gpurun_out/prof_lm_sort_$cfg.ncu-rep --page raw --csv > gpurun_out/prof_lm_sort_$cfg.raw.csv 2>/dev/null
rm -f gpurun_out/prof_lm_sort_$cfg.ncu-rep
echo done
