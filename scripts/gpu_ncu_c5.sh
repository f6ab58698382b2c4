set -u
OUT=gpurun_out; TAG=${1:-r2r}
make -s lib >/dev/null 2>&1
ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_c5_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-components > $OUT/ncu_c5_$TAG.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-components > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
