#!/bin/bash
# Exploration: fp64 latencies, upper bounds (no cold path / no fences), cluster sizes, per-round times.
OUT=gpurun_out
{
chmod +x tools/micro/fp64_latency; ./tools/micro/fp64_latency
bash tools/ab_variants.sh "" nocold nofence
for c in 8 6 5 4 2; do echo -n "C<=$c: "; MP_CLUSTER=$c timeout 60 python tools/profile_run.py --passes 6 | tail -2 | awk '{printf "%.3f ", $2*1000}'; echo; done
} > $OUT/explore.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_round -s 208 -c 52 --csv --log-file $OUT/rounds.csv \
    python tools/profile_run.py --passes 6 > $OUT/ncu_rounds.log 2>&1
echo done
