#!/bin/bash
# Peer-memory slab transport: mirror/flag unit tests, multi-process device slabs
# (ranks share one GPU; CUDA IPC works within a device), and the N=2 bench path.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "mirror or peer_flags or slabs_on_device" > gpurun_out/pytest_peer.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_peer.log
tail -15 gpurun_out/pytest_peer.log
for tr in peer nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus 2 --steps 30 --warmup 3 --dist-backend gloo --transport $tr --no-cpu --no-e2e > gpurun_out/bench_n2_$tr.json 2> gpurun_out/bench_n2_$tr.err
echo "n2 $tr rc=$?"; cat gpurun_out/bench_n2_$tr.json; grep -v OMP_NUM gpurun_out/bench_n2_$tr.err | grep -v '^\*' | tail -5
done
