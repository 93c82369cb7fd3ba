#!/bin/bash
# A/B of bench lines: each argument is "ENV=.. ENV2=..|bench args"; prints value/frac/ms.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/ab.jsonl
for item in "$@"; do
  envs=${item%%|*}; args=${item#*|}
  timeout 300 env $envs python bench.py --no-cpu --no-e2e $args 2>>gpurun_out/ab.err \
    | tee -a gpurun_out/ab.jsonl | python -c "import json,sys
try:
 d=json.loads(sys.stdin.read()); m=d.get('modes') or {}
 print('$envs | $args ->', d['value'], d['roofline']['frac'], d['plan'], d['ms_per_step'], 'other:', {k:v for k,v in m.items() if k!='fast_vs_exact'}, (m.get('fast_vs_exact') or {}).get('bitwise_equal'), d['clocks']['sm_mhz'], d['clocks']['reasons'])
except Exception as e: print('$envs | $args FAILED', e)"
done
