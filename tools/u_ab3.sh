#!/bin/bash
# Config 2/3 pass time per batch-size variant library (MP_BATCH = 4 / 6 for every shape) against the main library.
for cfg in 3 2; do
for v in "" u6 u4; do
  r=$(MP_LIB_VARIANT=$v python bench.py --config $cfg --no-cpu --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg variant '${v:-main}': $r ms/pass"
done; done
