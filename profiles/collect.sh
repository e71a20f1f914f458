#!/usr/bin/env bash
# Round profile collection (run on the GPU box under gpurun from the repo root):
#   gpurun --timeout 1800 -- 'bash profiles/collect.sh c2'
# Writes raw captures to gpurun_out/; profiles/summarize.py turns them into
# the committed summaries under profiles/.
set -u
cfg=${1:-c2}
export PYTHONPATH=$PWD:$PWD/tests
mkdir -p gpurun_out
# 1. the bench line itself (no profiler attached)
timeout 900 python bench.py --config "$cfg" > gpurun_out/bench_$cfg.json 2> gpurun_out/bench_$cfg.err
# 2. launch list of the same command (cold-cache, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_$cfg.csv \
  python bench.py --config "$cfg" --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
# 3. dram traffic of every local-moving launch of one Louvain run
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --clock-control none -k regex:'^lm_' --csv --log-file gpurun_out/move_traffic_$cfg.csv \
  python profiles/prof_run.py "$cfg" 1 > gpurun_out/move_traffic_$cfg.log 2>&1
# 4. full capture of the dominant local-moving kernels (first iteration of pass 0)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'^lm_p?sort' -c 6 \
  -o gpurun_out/prof_lm_sort_$cfg -f python profiles/prof_run.py "$cfg" 1 > gpurun_out/prof_lm_sort_$cfg.log 2>&1
echo done
