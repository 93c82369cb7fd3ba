#!/bin/bash
# Round evidence: gpu tests, smoke, bench lines for every config, reference arm,
# ncu launch lists (C3 default, C4) and one ncu --set full per dominant kernel.
cd "$(dirname "$0")/.."
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log; tail -2 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log; tail -2 $O/smoke.log
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"; cat $O/bench_c3.json
timeout 900 python bench.py --impl reference > $O/bench_c3_reference.json 2> $O/bench_c3_reference.err; echo "ref rc=$?"
for c in c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; echo "bench $c rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $O/launches_c3.csv python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e --no-mode-check > /dev/null 2>&1; echo "ncu c3 list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv --log-file $O/launches_c4.csv python bench.py --config c4 --steps 6 --warmup 3 --no-cpu --no-e2e --no-mode-check > /dev/null 2>&1; echo "ncu c4 list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tb3d_kernel -s 2 -c 1 -o $O/prof_c3_tb3d python bench.py --no-cpu --no-e2e --no-mode-check --steps 12 --warmup 3 > $O/ncu_c3.log 2>&1; echo "ncu c3 full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:box3d_kernel -s 2 -c 1 -o $O/prof_c4_box3d python bench.py --config c4 --no-cpu --no-e2e --no-mode-check --steps 6 --warmup 3 > $O/ncu_c4.log 2>&1; echo "ncu c4 full rc=$?"
