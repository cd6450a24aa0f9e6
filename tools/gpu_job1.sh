mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_large_tiles.py tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/pytest_r02m_b.log 2>&1; tail -5 gpurun_out/pytest_r02m_b.log
for cfg in 2 3 4 5; do
  r=$(python bench.py --config $cfg --no-cpu --steps 4 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('%.3f' % d['ms_per_step'])"); echo "config $cfg: $r ms/pass"
done
