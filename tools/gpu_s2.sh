set -u
OUT=gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x > $OUT/pytest_gpu_s2.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_s2.log
timeout 600 python bench.py > $OUT/bench_s2.json 2> $OUT/bench_s2.err; echo "bench rc=$?"; cat $OUT/bench_s2.json
for R in 5 25 45; do
  echo "== round $R"
  MP_LIB_VARIANT=tl MP_TL_ROUND=$R TL_CRIT=1 timeout 120 python tools/timeline.py --passes 4
  MP_LIB_VARIANT=tl MP_TL_ROUND=$R TL_SUMMARY=1 timeout 120 python tools/timeline.py --passes 4
done > $OUT/tl_s2.log 2>&1
MP_LIB_VARIANT=tl MP_TL_ROUND=25 timeout 120 python tools/timeline.py --passes 4 --dump $OUT/tl25.npy > $OUT/tl25_full.log 2>&1
echo done
