#!/bin/bash
# Config 4 (rounds of 2-CTA clusters in waves): slots per thread and batch size against the ring capacity.
run() { r=$(env "$@" python bench.py --config 4 --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config 4 $*: $r ms/pass"; }
run MP_LIB_VARIANT=knobs
run MP_LIB_VARIANT=knobs MP_SLOTS=3
run MP_LIB_VARIANT=knobs MP_SLOTS=4
run MP_LIB_VARIANT=u6
run MP_LIB_VARIANT=u6 MP_SLOTS=3
run MP_LIB_VARIANT=u4 MP_SLOTS=3
run MP_LIB_VARIANT=knobs MP_WAVE_C=3
run MP_LIB_VARIANT=knobs MP_WAVE_C=4
