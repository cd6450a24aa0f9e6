#!/bin/bash
# parity tests + A/B timing + cold-batch breakdown of round 25 (timeline build)
OUT=gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
bash tools/ab_variants.sh "$@"
MP_LIB_VARIANT=tl MP_TL_ROUND=25 TL_SUMMARY=1 timeout 120 python tools/timeline.py --passes 4 2>/dev/null
MP_LIB_VARIANT=tl MP_TL_ROUND=25 TL_CRIT=1 timeout 120 python tools/timeline.py --passes 4 2>/dev/null
} > $OUT/ab.log 2>&1
echo done
