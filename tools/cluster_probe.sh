for c in 1 8; do echo "== trace C=$c"; MP_CLUSTER=$c MP_LIB_VARIANT=trace python tools/trace_pass.py --passes 5; done
for v in "" nofence nocold; do for c in 1 4 8; do echo -n "variant=${v:-main} C=$c: "; MP_CLUSTER=$c MP_LIB_VARIANT=$v python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done; done
