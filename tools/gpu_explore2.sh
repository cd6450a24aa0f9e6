#!/bin/bash
OUT=gpurun_out
{
for v in tr trnc; do echo "== $v"; MP_LIB_VARIANT=$v timeout 120 python tools/trace_pass.py --passes 5; done
for R in 26 5; do echo "== tlnc round $R"; MP_LIB_VARIANT=tlnc MP_TL_ROUND=$R TL_CRIT=1 timeout 120 python tools/timeline.py --passes 4; done
} > $OUT/explore2.log 2>&1
MP_LIB_VARIANT=tlnc MP_TL_ROUND=26 timeout 120 python tools/timeline.py --passes 4 --dump $OUT/tlnc26.npy > /dev/null 2>&1
MP_LIB_VARIANT=tl MP_TL_ROUND=26 timeout 120 python tools/timeline.py --passes 4 --dump $OUT/tl26.npy > /dev/null 2>&1
echo done
