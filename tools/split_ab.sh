#!/bin/bash
# Hub band split (MP_HUB_RMAX = most rows of a band, MP_HUB_NWC compute warps; MP_NO_HUB_SPLIT: uniform bands) at config 3.
for v in "MP_HUB_RMAX=6" "MP_HUB_RMAX=6 MP_HUB_NWC=14" "MP_HUB_RMAX=6 MP_HUB_NWC=12"; do
env $v MP_VERBOSE=1 python -c "
from paper_1901_10084_b200 import instances
from paper_1901_10084_b200.solver import DeviceSession
s = DeviceSession(instances.config_instance(3), 'tiled', 40); s.close()" 2>&1 | grep -E "hub bands"
done
run() { r=$(env "$@" python bench.py --config 3 --no-cpu --steps 4 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config 3 $*: $r ms/pass"; }
run MP_HUB_RMAX=6
run MP_HUB_RMAX=6 MP_HUB_NWC=14
run MP_HUB_RMAX=6 MP_HUB_NWC=12
