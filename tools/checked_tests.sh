#!/bin/bash
# Checked build (MP_CHECKED device assertions; compute-sanitizer is closed on this pool):
# the GPU test suite, then every launch shape at two sizes, bitwise against the oracle.
OUT=gpurun_out/checked
mkdir -p $OUT
export MP_LIB_VARIANT=checked
timeout 2400 python -m pytest tests -m gpu -q -x > $OUT/pytest_checked.log 2>&1; echo "pytest (checked build) rc=$?"; tail -2 $OUT/pytest_checked.log
run() {  # label, n, env...
  label=$1; n=$2; shift 2
  env "$@" timeout 900 python tools/sanitize_run.py --n $n --passes 4 > $OUT/shape_${label}_n$n.log 2>&1
  echo "$label n=$n rc=$? $(grep -E 'bitwise|MP_ASSERT' $OUT/shape_${label}_n$n.log | head -2 | tr '\n' ' ')"
}
for n in 150 700; do
  run default $n MP_X=0
  run c1 $n MP_FORCE_C=1 MP_NO_DF=1
  run c2 $n MP_FORCE_C=2 MP_NO_DF=1
  run c2_u8 $n MP_FORCE_C=2 MP_NO_DF=1 MP_U=8
  run c8 $n MP_FORCE_C=8 MP_NO_DF=1
  run notma_c8 $n MP_FORCE_C=8 MP_NO_TMA=1 MP_NO_DF=1
  run waves $n MP_FORCE_C=2 MP_NO_DF=1 MP_CLUSTER=2
  run df_c2 $n MP_DF_C=2
  run df_c8 $n MP_DF_C=8
  run df_notma $n MP_DF_C=4 MP_NO_TMA=1
  run hub $n MP_X=0 MP_HUB_C=8
done
