#!/bin/bash
# FP64/FP32 pipe ceilings (tools/microbench) + bench lines carrying the arith roofline.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/fp
./tools/microbench/fp64_peak > gpurun_out/fp/fp_peaks.json 2> gpurun_out/fp/fp_peaks.err; echo "fp64_peak rc=$?"; cat gpurun_out/fp/fp_peaks.json
cp gpurun_out/fp/fp_peaks.json profiles/fp_peaks.json
timeout 600 python bench.py --no-cpu > gpurun_out/fp/bench_c3.json 2> gpurun_out/fp/bench_c3.err; echo "c3 rc=$?"; cat gpurun_out/fp/bench_c3.json; tail -3 gpurun_out/fp/bench_c3.err
timeout 600 python bench.py --config c4 --no-cpu --no-e2e > gpurun_out/fp/bench_c4.json 2> gpurun_out/fp/bench_c4.err; echo "c4 rc=$?"; cat gpurun_out/fp/bench_c4.json
