#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, tile-kernel DRAM bytes, full capture.
# Usage (on the GPU box): tools/gpu_round.sh <tag>
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json
# launch list of the bench command (short K)
python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/bench_short_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
# DRAM bytes + duration of every tile-kernel launch of pass 4 (config 2)
python tools/profile_run.py --passes 4 > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:tile_round -s 150 -c 50 --csv --log-file $OUT/tile_dram_$TAG.csv \
    python tools/profile_run.py --passes 4 > $OUT/ncu_dram_$TAG.log 2>&1; echo "ncu dram rc=$?"
# one full capture of the biggest round of pass 3
ncu --set full --clock-control none --import-source on -k regex:tile_round -s 130 -c 1 \
    -o $OUT/prof_tile_$TAG python tools/profile_run.py --passes 3 > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
