#!/bin/bash
# Pass time per (MP_MIN_C, MP_LANES) of the per-round launches: fewer lanes per warp spread a hub tile's exact
# steps over more warps (the dataflow launch keeps its own shape; MP_DF_LANES).
for cfg in 2 3; do
for v in "MP_X=0" "MP_MIN_C=8" "MP_MIN_C=8 MP_LANES=15" "MP_MIN_C=8 MP_LANES=20" "MP_MIN_C=7 MP_LANES=18" "MP_MIN_C=6 MP_LANES=21"; do
  r=$(env $v python bench.py --config $cfg --no-cpu --steps 4 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
  echo "config $cfg $v: $r ms/pass"
done
done
