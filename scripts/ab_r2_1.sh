set -u
ROUNDS=2 bash scripts/ab.sh build/ab/base.so build/ab/dedup.so build/ab/sched.so
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/base.so build/ab/dedup.so build/ab/sched.so
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c5ab_base.npy'); 
for n in ('dedup','sched'):
    b=np.load(f'gpurun_out/c5ab_{n}.npy')
    same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all()
    print(n, 'bit-identical summaries' if same else 'DIFFERENT')
PY
