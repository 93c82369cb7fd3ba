#!/bin/bash
# Sweep + one ncu --set full capture per requested tag.
#   SWEEP="c3:--fused 3 --mode fast;c3:--fused 3" NCU="tag|regex|bench args;..." tools/gpu_prof.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
IFS=';' read -ra S <<< "$SWEEP"
for item in "${S[@]}"; do
  [ -z "$item" ] && continue
  cfg=${item%%:*}; args=${item#*:}
  timeout 300 python bench.py --no-cpu --no-e2e --config $cfg $args 2>>gpurun_out/sweep.err | tee -a gpurun_out/sweep.jsonl | python -c "import json,sys
try:
 d=json.loads(sys.stdin.read()); print('$cfg $args', d['value'], d['roofline']['frac'], d['plan']['engine'], d['plan']['fused_steps'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$cfg $args FAILED', e)"
done
IFS=';' read -ra N <<< "$NCU"
for item in "${N[@]}"; do
  [ -z "$item" ] && continue
  IFS='|' read -r tag kre args <<< "$item"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
    -o gpurun_out/prof_$tag python bench.py --no-cpu --no-e2e --steps 12 --warmup 3 $args \
    > gpurun_out/ncu_$tag.log 2>&1
  echo "ncu $tag rc=$?"; tail -2 gpurun_out/ncu_$tag.log
done
