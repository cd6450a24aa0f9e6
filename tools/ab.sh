#!/bin/bash
# A/B timing of env variants on config 2 (pass 5 device time, 3 repeats)
run() { for r in 1 2 3; do env "$@" python tools/profile_run.py --passes 5 | tail -1 | awk '{printf "%.2f ", $2*1000}'; done; echo " <- $*"; }
for v in "$@"; do run $v; done
