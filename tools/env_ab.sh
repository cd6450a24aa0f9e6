#!/bin/bash
# Pass times of one config under several environment variants.
# Usage: tools/env_ab.sh <config> <passes> "<VAR=v VAR2=w>" ...
C=$1; P=$2; shift 2
for v in "$@"; do
  echo "== config $C env: $v"
  env $v timeout 600 python tools/profile_run.py --config $C --passes $P 2>&1 | grep -v Warn | grep -v "^\[mp\] pool" | tail -$((P+1)) | cut -c1-400
done
