#!/bin/bash
OUT=gpurun_out
MP_LIB_VARIANT=tlnc MP_TL_ROUND=26 timeout 120 python tools/timeline.py --passes 4 --dump $OUT/tlnc26p.npy > $OUT/explore3.log 2>&1
echo done
