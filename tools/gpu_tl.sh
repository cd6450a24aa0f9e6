#!/bin/bash
# cold-batch summary + critical-band summary of a few rounds (timeline build)
OUT=gpurun_out
for R in "$@"; do
  echo "== round $R"
  MP_LIB_VARIANT=tl MP_TL_ROUND=$R TL_SUMMARY=1 timeout 120 python tools/timeline.py --passes 4 2>/dev/null
  MP_LIB_VARIANT=tl MP_TL_ROUND=$R TL_CRIT=1 timeout 120 python tools/timeline.py --passes 4 2>/dev/null
  MP_LIB_VARIANT=tl MP_TL_ROUND=$R timeout 120 python tools/timeline.py --passes 4 --dump $OUT/tl$R.npy >/dev/null 2>&1
done > $OUT/tl.log 2>&1
