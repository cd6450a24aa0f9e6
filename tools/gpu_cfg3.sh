#!/bin/bash
# config 3 pass time (ms, passes 3-4) for variants / env settings
{
for v in "$@"; do echo -n "cfg3 $v: "; env $v timeout 300 python tools/profile_run.py --config 3 --passes 4 | tail -2 | awk '{printf "%.2f ", $2*1000}'; echo; done
} > gpurun_out/cfg3.log 2>&1
