#!/bin/bash
# pass time (ms, passes 5-6 of config 2): variants x cluster size x slots x ring width
for v in "" nostag; do for c in 8 4; do for sl in 1 2; do for w in 256 512; do
  echo -n "v=${v:-main} C=$c S>=$sl W<=$w: "; MP_LIB_VARIANT=$v MP_CLUSTER=$c MP_SLOTS=$sl MP_RING_W=$w timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo
done; done; done; done
