#!/bin/bash
# Pass time per forced cluster size (MP_FORCE_C: one C for every round, in waves when the
# round's clusters do not all fit) vs the default plan.  Usage: tools/force_c.sh <config> <passes>
C=${1:-5}; P=${2:-3}
for fc in "" 2 4 8; do
  echo "== MP_FORCE_C=$fc"
  MP_FORCE_C=$fc timeout 600 python tools/profile_run.py --config $C --passes $P 2>&1 | grep -v Warn | tail -$P
done
