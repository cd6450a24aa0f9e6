#!/bin/bash
# A/B timing of library variants (MP_LIB_VARIANT) on config 2: last 2 of 6 passes, ms
# usage: tools/ab_variants.sh "" old nocold ...   (env such as MP_CLUSTER passes through)
vs=("$@"); [ ${#vs[@]} -eq 0 ] && vs=("" old)
for v in "${vs[@]}"; do
  echo -n "variant=${v:-main}: "; MP_LIB_VARIANT=$v python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo
done
