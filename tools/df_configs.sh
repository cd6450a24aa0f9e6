#!/bin/bash
# Pass times per BASELINE config with and without the dataflow launch (MP_NO_DF).
for cfg in 2 3 4 5; do
  st=6; [ $cfg -ge 4 ] && st=2
  for v in "MP_X=0" "MP_NO_DF=1"; do
    r=$(env $v timeout 900 python bench.py --config $cfg --no-cpu --steps $st --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])")
    echo "config $cfg $v: $r ms/pass"
  done
done
