#!/bin/bash
# A/B of the late-pass options: serial bins (LVN_FORK_VERTS_LOG2=0), forked
# bins (default), forked bins + captured while-loop passes
# (LVN_GRAPH_VERTS_LOG2=22).  bash profiles/graph_ab.sh [configs...]
cd "$(dirname "$0")/.."
export PYTHONPATH=$PWD
for c in ${@:-c1 c4 c2}; do
  for mode in "LVN_FORK_VERTS_LOG2=0" "DEFAULT=1" "LVN_GRAPH_VERTS_LOG2=22"; do
    echo "== $c $mode"
    env $mode timeout 300 python profiles/prof_run.py $c 5 2>&1 | tail -3 | cut -c1-330
  done
done
