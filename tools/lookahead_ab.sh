#!/bin/bash
# Ring blocks loaded ahead of the fastest warp (MP_LOOKAHEAD builds la6 / la8 against the main library's 4).
for cfg in 2 3 4; do
  for v in "" la6 la8; do
    r=$(MP_LIB_VARIANT=$v python bench.py --config $cfg --no-cpu --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
    echo "config $cfg variant '${v:-main}': $r ms/pass"
  done
done
