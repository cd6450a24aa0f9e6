#!/bin/bash
# config 5 pass times (s, passes 1-2) under env settings
for v in "$@"; do echo "== $v"; env $v timeout 600 python tools/profile_run.py --config 5 --passes 2; done > gpurun_out/cfg5.log 2>&1
