#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, tile-kernel DRAM bytes, full capture.
# Usage (on the GPU box): tools/gpu_round.sh <tag> [config]   (default config 3, the bench workload)
set -u
TAG=${1:-r02}
CFG=${2:-3}
OUT=gpurun_out
mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py --config $CFG > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json
# launch list of the bench command (short K)
python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu > $OUT/bench_short_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu > $OUT/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
# DRAM bytes + duration of every tile-kernel launch of pass 4
NR=$(python -c "from paper_1901_10084_b200 import schedule, instances as I; n=I.CONFIGS[$CFG].n; print(sum(1 for r in schedule.tiled_rounds(n, 40) if r.units))")
python tools/profile_run.py --config $CFG --passes 4 > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:tile_round -s $((3 * NR)) -c $NR --csv --log-file $OUT/tile_dram_$TAG.csv \
    python tools/profile_run.py --config $CFG --passes 4 > $OUT/ncu_dram_$TAG.log 2>&1; echo "ncu dram rc=$?"
# one full capture of a mid-pass round of pass 3
ncu --set full --clock-control none --import-source on -k regex:tile_round -s $((2 * NR + NR / 2)) -c 1 \
    -o $OUT/prof_tile_$TAG python tools/profile_run.py --config $CFG --passes 3 > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
