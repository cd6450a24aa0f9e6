{ for w in 512 256; do echo -n "W=$w: "; MP_RING_W=$w timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done
  for w in 512 256; do echo -n "nocold W=$w: "; MP_LIB_VARIANT=nocold MP_RING_W=$w timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done
  for w in 512 256; do echo -n "cfg3 W=$w: "; MP_RING_W=$w timeout 200 python tools/profile_run.py --config 3 --passes 4 | tail -2 | awk '{printf "%.2f ", $2*1000}'; echo; done
} > gpurun_out/ab.log 2>&1
