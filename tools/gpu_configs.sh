#!/bin/bash
# Bench lines for the larger BASELINE configs (2, 3, 4, 5) at N=1, no CPU leg.
# Usage (on the GPU box): tools/gpu_configs.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
for c in 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu > $OUT/bench_cfg${c}_$TAG.json 2> $OUT/bench_cfg${c}_$TAG.err
  echo "config $c rc=$?"; cat $OUT/bench_cfg${c}_$TAG.json
done
