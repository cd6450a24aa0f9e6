#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list, tile-kernel DRAM bytes, full captures.
# Usage (on the GPU box): tools/gpu_round.sh <tag> [config]   (default config 3, the bench workload)
set -u
TAG=${1:-r02}
CFG=${2:-3}
OUT=gpurun_out
mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
timeout 1200 python bench.py --config $CFG > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json
timeout 900 python bench.py --config $CFG --impl reference > $OUT/bench_reference_$TAG.json 2> $OUT/bench_reference_$TAG.err; echo "reference rc=$?"; cat $OUT/bench_reference_$TAG.json
# launch list of the bench command (short K)
python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu > $OUT/bench_short_$TAG.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu > $OUT/ncu_launches_$TAG.log 2>&1; echo "ncu launches rc=$?"
# tile-kernel launches per pass: the first family's rounds, one per round, plus the dataflow launch
NR=$(python -c "
from paper_1901_10084_b200 import schedule, instances as I
rs=[r for r in schedule.tiled_rounds(I.CONFIGS[$CFG].n, 40) if r.units]
r0=next(i for i,r in enumerate(rs) if r.units[0].x >= 1)
print(r0 + 1)")
echo "tile launches per pass: $NR"
# DRAM bytes + duration of every tile-kernel launch of pass 4
python tools/profile_run.py --config $CFG --passes 4 > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,smsp__inst_executed.sum \
    --clock-control none -k regex:tile_round -s $((3 * NR)) -c $NR --csv --log-file $OUT/tile_dram_$TAG.csv \
    python tools/profile_run.py --config $CFG --passes 4 > $OUT/ncu_dram_$TAG.log 2>&1; echo "ncu dram rc=$?"
# full captures of pass 3: a first-family round (round 10: hub rows in its longest tile) and the dataflow launch
ncu --set full --clock-control none --import-source on -k regex:tile_round -s $((2 * NR + 10)) -c 1 \
    -o $OUT/prof_tile_$TAG python tools/profile_run.py --config $CFG --passes 3 > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:tile_round -s $((3 * NR - 1)) -c 1 \
    -o $OUT/prof_df_$TAG python tools/profile_run.py --config $CFG --passes 3 > $OUT/ncu_full_df_$TAG.log 2>&1; echo "ncu full df rc=$?"
