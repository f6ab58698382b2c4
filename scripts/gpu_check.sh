#!/usr/bin/env bash
# One GPU round trip: parity tests, smoke, bench, ncu launch list + full capture.
# Usage (from the repo root, under gpurun): bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)" > $OUT/lscpu_$TAG.txt 2>&1
make -s lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke_$TAG.log
ARROW_BENCH_DUMP=$OUT/summaries_$TAG.npy timeout 900 python bench.py --steps 3 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; cat $OUT/bench_$TAG.json; tail -3 $OUT/bench_$TAG.err
if [ "${SKIP_NCU:-0}" != "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $OUT/ncu_launch_bench_$TAG.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 $OUT/ncu_full_$TAG.log
fi
