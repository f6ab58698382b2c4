set -u
ROUNDS=2 bash scripts/ab.sh build/ab/base.so build/ab/sched.so build/ab/cur.so
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/sched.so build/ab/cur.so build/ab/cur_tp2.so build/ab/cur_tp4.so
ARROW_SIM_LIB=build/ab/cur.so ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o gpurun_out/prof_c5_r2d -f \
  python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-components > gpurun_out/ncu_c5_r2d.log 2>&1; echo "ncu rc=$?"
