set -u
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/lean.so build/ab/slim.so
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c5ab_lean.npy'); b=np.load('gpurun_out/c5ab_slim.npy')
same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all() and (a['stall_time'].view('u8')==b['stall_time'].view('u8')).all()
print('slim vs lean:', 'bit-identical summaries' if same else 'DIFFERENT')
print('steps serial %.3g -> %.3g, parallel %.3g -> %.3g' % (a['n_serial_steps'].sum(), b['n_serial_steps'].sum(), a['n_parallel_steps'].sum(), b['n_parallel_steps'].sum()))
PY
for W in c3 c4 c2; do for L in lean slim; do ARROW_SIM_LIB=build/ab/$L.so python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W $L %.1f ms' % d['ms_per_step'])"; done; done
