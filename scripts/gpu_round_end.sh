#!/usr/bin/env bash
# Round-end evidence run: GPU tests, smoke, default bench (C5) + reference arm,
# C2-C4 lines, ncu --set full of a 4 096-scenario C5 launch, launch list of the bench command.
set -u
TAG=${1:-final}; OUT=gpurun_out
mkdir -p $OUT
bash scripts/gpu_final.sh $TAG
NCU_C4=0 true
ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_c5_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-components > $OUT/ncu_c5_$TAG.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-components > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
