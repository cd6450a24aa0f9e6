#!/bin/bash
# One short bench line per config 2, 3, 4 (no CPU leg): pass time after a kernel change.
for cfg in 2 3 4; do
  r=$(python bench.py --config $cfg --no-cpu --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg: $r ms/pass"
done
