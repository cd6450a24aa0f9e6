#!/bin/bash
OUT=gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in "MP_VERBOSE=1" "MP_WR_PITCH_W=1" "MP_WK_PITCH_B=1" "MP_WR_PITCH_W=1 MP_WK_PITCH_B=1"; do echo -n "$v: "; env $v timeout 60 python tools/profile_run.py --passes 6 2>&1 | tail -3 | awk '{printf "%s ", $0}'; echo; done
} > $OUT/ab.log 2>&1
bash tools/gpu_cfg3.sh MP_VERBOSE=1 MP_WR_PITCH_W=1; cat $OUT/cfg3.log >> $OUT/ab.log
