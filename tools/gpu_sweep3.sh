#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/sweep.jsonl
run() { timeout 300 env $1 python bench.py --no-cpu --no-e2e ${@:2} 2>>gpurun_out/sweep.err | tee -a gpurun_out/sweep.jsonl | python -c "import json,sys
try:
 d=json.loads(sys.stdin.read()); print('$1 ${*:2}', d['value'], d['roofline']['frac'], d['config']['engine'], d['config']['fused_steps'], d['ms_per_step'], d['clocks']['sm_mhz'])
except Exception: print('$1 ${*:2} FAILED')"; }
for k in 1 2 3; do run X=1 --fused $k; run X=1 --fused $k --mode fast; done
