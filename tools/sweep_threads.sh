#!/bin/bash
# quick tuning sweep of CTA thread counts on config 2
for t in 512 416 320; do
  echo "MP_CTA_THREADS=$t"
  MP_CTA_THREADS=$t python tools/profile_run.py --passes 6 | tail -2
done
