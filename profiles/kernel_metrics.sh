#!/usr/bin/env bash
# Per-launch counters of the local-moving and aggregation kernels of one C2 run
# (ncu, one pass per metric group; run on the GPU box from the repo root).
#   bash profiles/kernel_metrics.sh <config> <out.csv> [kernel-regex]
set -u
cfg=${1:-c2}; out=${2:-gpurun_out/kmetrics.csv}; rx=${3:-'^(lm_|ag_)'}
export PYTHONPATH=$PWD:$PWD/tests
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
M=$M,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size
M=$M,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_membar_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_drain_per_issue_active.ratio
M=$M,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio
M=$M,smsp__thread_inst_executed_per_inst_executed.ratio
timeout 900 ncu --metrics $M --clock-control none -k regex:"$rx" --csv --log-file "$out" \
  python profiles/prof_run.py "$cfg" 1 > "${out%.csv}.log" 2>&1
