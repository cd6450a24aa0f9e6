#!/bin/bash
# Rounds of up to MP_MIN_C_CNT tiles get >= 6 CTAs per tile (default 55 = 3/8 of the SMs): re-check after the U = 4 fix of the 2-CTA shape.
run() { cfg=$1; shift; r=$(env MP_LIB_VARIANT=knobs "$@" python bench.py --config $cfg --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg $*: $r ms/pass"; }
for c in 40 48 55 64 72 90; do run 4 MP_MIN_C_CNT=$c; done
for c in 40 55 72 100; do run 5 MP_MIN_C_CNT=$c; done
