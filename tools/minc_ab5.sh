#!/bin/bash
# Config 5 (hub instance): larger rounds still gain from >= 6 CTAs per tile (hub shape).
run() { cfg=$1; shift; r=$(env MP_LIB_VARIANT=knobs "$@" python bench.py --config $cfg --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg $*: $r ms/pass"; }
for c in 100 125 150 180 230; do run 5 MP_MIN_C_CNT=$c; done
