#!/bin/bash
# Pass times per wave cluster size (MP_WAVE_C: C for rounds whose clusters do not all fit;
# 1 = the old one-CTA-per-tile fallback).  Usage: tools/wave_c.sh <config> <passes> [values]
C=${1:-5}; P=${2:-3}; shift 2
for w in ${@:-1 2 3}; do
  echo "== config $C MP_WAVE_C=$w"
  MP_WAVE_C=$w timeout 600 python tools/profile_run.py --config $C --passes $P 2>&1 | grep -v Warn | tail -$P
done
