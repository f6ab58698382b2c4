set -u
TAG=r2a
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
lscpu > $OUT/lscpu_$TAG.txt 2>&1
make -s lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -5 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -3 $OUT/smoke_$TAG.log
ARROW_BENCH_DUMP=$OUT/c5sum_$TAG.npy timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline --no-components > $OUT/bench_c5_$TAG.json 2> $OUT/bench_c5_$TAG.err; echo "bench c5 rc=$?"; cat $OUT/bench_c5_$TAG.json; tail -3 $OUT/bench_c5_$TAG.err
ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_c5_$TAG -f \
  python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-components > $OUT/ncu_full_c5_$TAG.log 2>&1; echo "ncu full rc=$?"; tail -3 $OUT/ncu_full_c5_$TAG.log
