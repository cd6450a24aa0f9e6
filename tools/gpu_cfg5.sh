#!/bin/bash
# config 5 pass times (s, passes 1-3) for variants
for v in "$@"; do echo "== ${v:-main}"; MP_LIB_VARIANT=$v timeout 600 python tools/profile_run.py --config 5 --passes 3; done > gpurun_out/cfg5.log 2>&1
