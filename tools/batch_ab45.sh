#!/bin/bash
# Pass times at configs 4 and 5 per library variant (batch sizes u2/u4 vs the main library's U = 8).
for cfg in 4 5; do
  for v in "" $@; do
    r=$(MP_LIB_VARIANT=$v python bench.py --config $cfg --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
    echo "config $cfg variant '${v:-main}': $r ms/pass"
  done
done
