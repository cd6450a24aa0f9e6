#!/bin/bash
# A/B of the dataflow launch's cluster size (MP_DF_C) and of no dataflow (MP_NO_DF): pass times at configs 2 and 3.
for cfg in 2 3; do
  for v in "MP_NO_DF=1" "MP_DF_C=2" "MP_DF_C=3" "MP_DF_C=4" "MP_DF_C=6" "MP_DF_C=8"; do
    r=$(env $v python bench.py --config $cfg --no-cpu --steps 6 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
    echo "config $cfg $v: $r ms/pass"
  done
done
