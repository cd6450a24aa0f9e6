#!/bin/bash
# parity tests + A/B timing (config 2) of variants, with env overrides applied to all
OUT=gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/ab_variants.sh "$@"
echo -n "MP_NO_TMA main: "; MP_NO_TMA=1 timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo
} > $OUT/ab.log 2>&1
echo done
