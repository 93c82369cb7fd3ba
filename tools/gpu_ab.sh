#!/bin/bash
# A/B of engine variants selected by environment: VARIANTS="name:ENV=val ENV2=val;..."
#   SWEEP as in gpu_prof.sh; TESTS = pytest -k expression run once per variant.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab.txt
IFS=';' read -ra V <<< "$VARIANTS"
for v in "${V[@]}"; do
  name=${v%%:*}; envs=${v#*:}
  if [ -n "$TESTS" ]; then
    env $envs timeout 600 python -m pytest tests -m gpu -x -q -k "$TESTS" > gpurun_out/ab_tests_$name.log 2>&1
    echo "$name tests: $(tail -1 gpurun_out/ab_tests_$name.log)" | tee -a gpurun_out/ab.txt
  fi
  IFS=',' read -ra S <<< "$SWEEP"
  for item in "${S[@]}"; do
    cfg=${item%%:*}; args=${item#*:}
    env $envs timeout 300 python bench.py --no-cpu --no-e2e --config $cfg $args 2>>gpurun_out/ab.err | python -c "import json,sys
try:
 d=json.loads(sys.stdin.read()); print('$name $cfg $args', d['value'], d['roofline']['frac'], d['config']['fused_steps'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$name $cfg $args FAILED', e)" | tee -a gpurun_out/ab.txt
  done
done
