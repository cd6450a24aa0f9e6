#!/bin/bash
# pass time (config 2, last 2 of 6 passes, ms) by maximum cluster size
for c in 8 7 6 5 4; do echo -n "C<=$c: "; MP_CLUSTER=$c timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done > gpurun_out/ab.log 2>&1
