timeout 900 python -m pytest tests/test_gpu_golden_full.py tests/test_gpu_fullsize.py -m gpu -x -q -k "config5 or config4 or config3_passes" 2>&1 | tail -3
for cfg in 5 3; do r=$(python bench.py --config $cfg --no-cpu --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg: $r ms/pass"; done
