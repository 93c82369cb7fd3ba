#!/bin/bash
# Range sweeps + slab runner (several ranks sharing the GPU over gloo) + the N>1 bench path.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "sweep_range or slabs_on_device" > gpurun_out/pytest_slab.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_slab.log
tail -5 gpurun_out/pytest_slab.log
for ov in "" "--no-overlap"; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 30 --warmup 3 --dist-backend gloo --no-cpu --no-e2e $ov > gpurun_out/bench_n2_gloo$ov.json 2> gpurun_out/bench_n2_gloo$ov.err
echo "n2 gloo $ov rc=$?"; cat gpurun_out/bench_n2_gloo$ov.json; tail -3 gpurun_out/bench_n2_gloo$ov.err
done
