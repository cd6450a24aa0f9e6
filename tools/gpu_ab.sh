#!/bin/bash
# parity tests + A/B timing of config 2 (last 2 of 6 passes, ms) for the given variants
OUT=gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/ab_variants.sh "$@"
} > $OUT/ab.log 2>&1
echo done
