#!/bin/bash
# config 2 pass time (ms, last 2 of 6 passes) under env settings / variants
for v in "$@"; do echo -n "$v: "; env $v timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done > gpurun_out/ab.log 2>&1
