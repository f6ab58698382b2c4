set -u
ROUNDS=2 bash scripts/ab.sh build/ab/sched.so build/ab/unified.so
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/sched.so build/ab/unified.so
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c5ab_sched.npy'); b=np.load('gpurun_out/c5ab_unified.npy')
same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all()
print('unified vs sched:', 'bit-identical summaries' if same else 'DIFFERENT')
PY
ARROW_SIM_LIB=build/ab/unified.so ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o gpurun_out/prof_c5_r2c -f \
  python bench.py --workload c5 --steps 1 --warmup 0 --no-cpu-baseline --no-components > gpurun_out/ncu_c5_r2c.log 2>&1; echo "ncu rc=$?"
