#!/bin/bash
# Driver-style bench lines for every BASELINE config (cpu_baseline, e2e,
# modes, roofline), the reference arm for each (REF=0 skips them), and the
# N=2 slab path on the one visible GPU.  Outputs -> gpurun_out/lines/
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/lines
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 10 \
    > gpurun_out/lines/bench_$c.json 2> gpurun_out/lines/bench_$c.err
  echo "$c rc=$? $(head -c 200 gpurun_out/lines/bench_$c.json)"
  if [ "${REF:-1}" != 0 ]; then
    timeout 600 python bench.py --impl reference --config $c --steps ${STEPS:-20} --warmup 10 \
      > gpurun_out/lines/reference_$c.json 2> gpurun_out/lines/reference_$c.err
    echo "$c ref rc=$?"
  fi
done
timeout 600 python bench.py --gpus 2 --share-devices --steps 60 --warmup 10 \
  > gpurun_out/lines/bench_c3_n2_shared.json 2> gpurun_out/lines/bench_c3_n2_shared.err
echo "n2 rc=$?"
