#!/bin/bash
# config 3 (n=4000) pass time (ms) under cluster-size caps
for c in 8 6 4 2 1; do
  echo -n "cfg3 C<=$c: "; MP_CLUSTER=$c CFG=3 timeout 120 python tools/phase_time.py | tail -1
done
