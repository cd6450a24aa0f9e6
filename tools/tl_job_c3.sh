set -x
for spec in "0 1" "0 0" "40 0" "40 1" "10 1"; do
  set -- $spec
  MP_LIB_VARIANT=tl MP_TL_ROUND=$1 MP_TL_TILE=$2 TL_SUMMARY=1 python tools/timeline.py --config 3 --passes 4 > gpurun_out/tl_c3_r$1_t$2_sum.log 2>&1
  MP_LIB_VARIANT=tl MP_TL_ROUND=$1 MP_TL_TILE=$2 python tools/timeline.py --config 3 --passes 4 --dump gpurun_out/tl_c3_r$1_t$2.npy > gpurun_out/tl_c3_r$1_t$2.log 2>&1
done
