#!/bin/bash
# Quick GPU check: GPU tests (optionally a -k filter), config-3 bench (no CPU leg), per-tile times.
# Usage (on the GPU box): tools/gpu_quick.sh <tag> [pytest -k expr]
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
if [ -n "$2" ]; then K=(-k "$2"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -q -x "${K[@]}" > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_$TAG.log
timeout 600 python bench.py --config 3 --no-cpu --steps 10 > $OUT/bench3_$TAG.json 2> $OUT/bench3_$TAG.err; echo "bench3 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench3_$TAG.json')); print('config3', d['ms_per_step'], 'ms/pass', d['value'])"
timeout 600 python bench.py --config 2 --no-cpu --steps 20 > $OUT/bench2_$TAG.json 2> $OUT/bench2_$TAG.err; echo "bench2 rc=$?"
python -c "import json; d=json.load(open('$OUT/bench2_$TAG.json')); print('config2', d['ms_per_step'], 'ms/pass', d['value'])"
if [ -f paper_1901_10084_b200/_lib/libmetricproj_b200_tt.so ]; then
  MP_LIB_VARIANT=tt timeout 300 python tools/tile_times.py --config 3 --passes 4 --show 12 > $OUT/tt3_$TAG.log 2>&1; tail -1 $OUT/tt3_$TAG.log
fi
