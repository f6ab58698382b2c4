set -u
ROUNDS=2 bash scripts/ab.sh build/ab/cur.so build/ab/sm.so
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/cur.so build/ab/sm.so
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c5ab_cur.npy'); b=np.load('gpurun_out/c5ab_sm.npy')
same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all()
print('sm vs cur:', 'bit-identical summaries' if same else 'DIFFERENT')
PY
