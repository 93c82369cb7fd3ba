#!/bin/bash
# ncu --set full of the top kernel for one bench config.
#   tools/ncu_capture.sh <tag> <kernel-regex> <bench args...>
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
tag=$1; kre=$2; shift 2
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 2 -c 1 \
  -o gpurun_out/prof_$tag python bench.py --no-cpu --no-e2e --no-mode-check --steps 12 --warmup 3 "$@" \
  > gpurun_out/ncu_$tag.log 2>&1
echo "ncu $tag rc=$?"; tail -3 gpurun_out/ncu_$tag.log
