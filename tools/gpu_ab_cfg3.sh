OUT=gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
bash tools/ab_variants.sh "" u4
for v in "" u4; do echo -n "cfg3 ${v:-main}: "; MP_LIB_VARIANT=$v timeout 200 python tools/profile_run.py --config 3 --passes 4 | tail -2 | awk '{printf "%.2f ", $2*1000}'; echo; done
} > $OUT/ab.log 2>&1
