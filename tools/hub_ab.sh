#!/bin/bash
# Config-3 pass time per hub launch shape (MP_HUB_C / MP_HUB_LANES, the MP_CMAX=16 build for C > 8) and dataflow lanes.
run() { r=$(env "$@" python bench.py --config 3 --no-cpu --steps 4 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config 3 $*: $r ms/pass"; }
run MP_X=0
run MP_HUB_LANES=10
run MP_HUB_LANES=20
run MP_LIB_VARIANT=c16 MP_HUB_C=8
run MP_LIB_VARIANT=c16 MP_HUB_C=10
run MP_LIB_VARIANT=c16 MP_HUB_C=12
run MP_LIB_VARIANT=c16 MP_HUB_C=14
run MP_LIB_VARIANT=c16 MP_HUB_C=16
run MP_DF_LANES=10
run MP_DF_LANES=20
run MP_DF_C=3
