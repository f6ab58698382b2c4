set -u
for i in 1 2; do for L in ipl2_3 ipl2_2; do ARROW_SIM_LIB=build/ab/$L.so ARROW_BENCH_DUMP=gpurun_out/c4_$L.npy python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $L %.1f ms %.4g req/s' % (d['ms_per_step'], d['value']))"; done; done
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c4_ipl2_3.npy'); b=np.load('gpurun_out/c4_ipl2_2.npy')
same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all()
print('ipl2_2 vs ipl2_3 (C4):', 'bit-identical summaries' if same else 'DIFFERENT')
PY
