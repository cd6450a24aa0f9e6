#!/bin/bash
# Pass times at configs 2 and 3 per library variant (MP_LIB_VARIANT, e.g. batch sizes u4/u6/u12).
for cfg in 2 3; do
  for v in "" $@; do
    r=$(MP_LIB_VARIANT=$v python bench.py --config $cfg --no-cpu --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
    echo "config $cfg variant '${v:-main}': $r ms/pass"
  done
done
