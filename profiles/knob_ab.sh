#!/usr/bin/env bash
# A/B of an environment knob on bench.py (device-resident leg only), e.g.
#   gpurun -- 'bash profiles/knob_ab.sh LVN_SORT16 "0 1 3 0" c5 c3 c2'
# One JSON summary per run in gpurun_out/knob_ab.txt.
set -u
knob=$1; vals=$2; shift 2
export PYTHONPATH=$PWD
mkdir -p gpurun_out
for cfg in "$@"; do
  for v in $vals; do
    env "$knob=$v" timeout 600 python bench.py --config "$cfg" --steps 5 --warmup 3 --no-e2e --no-cpu-baseline \
      2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'knob':'$knob','val':'$v','cfg':'$cfg','Gedges':round(d['value']/1e9,3),'ms':round(d['ms_per_step'],2),
 'move_ms':round(d['kernel_seconds']['move']*1e3,2),'Q':round(d['modularity'],5),'step_ms':d['step_ms'],'iters':d['iterations_per_pass']}))
" >> gpurun_out/knob_ab.txt 2>&1
  done
done
