#!/bin/bash
OUT=gpurun_out
{
for p in 3 2 4 6 8; do echo -n "NPW=$p: "; MP_PRODUCERS=$p timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done
for p in 3 6; do echo -n "nocold NPW=$p: "; MP_LIB_VARIANT=nocold MP_PRODUCERS=$p timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done
} > $OUT/explore4.log 2>&1
echo done
