#!/bin/bash
# First GPU pass: parity tests, smoke, bench, launch list.  Outputs -> gpurun_out/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
cat gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"
cat gpurun_out/bench_c3.json; tail -5 gpurun_out/bench_c3.err
for c in c1 c2; do timeout 300 python bench.py --config $c --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; cat gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1; echo "ncu rc=$?"
