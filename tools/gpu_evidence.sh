#!/bin/bash
# Round evidence on one B200: sanitizer logs, per-config launch lists with
# DRAM bytes (-> profiles/ncu_traffic.json), and ncu --set full captures.
#   CFGS="c1 c2 c3 c4 c5" FULL="c3|tb3d_kernel;c1|stream2d" SAN=1 tools/gpu_evidence.sh
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
if [ -n "$SAN" ]; then
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_engines.py \
      > gpurun_out/sanitize_$tool.log 2>&1
    echo "sanitize $tool rc=$?"; tail -2 gpurun_out/sanitize_$tool.log
  done
fi
for c in $CFGS; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 60 --csv --log-file gpurun_out/launches_$c.csv \
    python bench.py --config $c --no-cpu --no-e2e --no-mode-check --steps 12 --warmup 3 \
    > gpurun_out/launches_$c.log 2>&1
  echo "launches $c rc=$?"
done
IFS=';' read -ra N <<< "$FULL"
for item in "${N[@]}"; do
  [ -z "$item" ] && continue
  IFS='|' read -r c kre <<< "$item"
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
    -o gpurun_out/prof_$c python bench.py --config $c --no-cpu --no-e2e --no-mode-check \
    --steps 12 --warmup 3 > gpurun_out/ncu_$c.log 2>&1
  echo "ncu $c rc=$?"; tail -2 gpurun_out/ncu_$c.log
  # summarise on the box (the reports themselves are too large to bring back)
  python tools/ncu_summary.py gpurun_out/prof_$c.ncu-rep > gpurun_out/ncu_${c}_summary.txt 2>&1
  ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass \
    > gpurun_out/ncu_${c}_sass.csv 2>/dev/null
  ncu -i gpurun_out/prof_$c.ncu-rep --page raw --csv > gpurun_out/ncu_${c}_raw.csv 2>/dev/null
  gzip -f gpurun_out/ncu_${c}_sass.csv
  rm -f gpurun_out/prof_$c.ncu-rep
done
for c in $CFGS; do
  python tools/launch_summary.py gpurun_out/launches_$c.csv > gpurun_out/launches_${c}_summary.txt 2>&1
done
