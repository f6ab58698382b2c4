set -u
# occupancy: 3 vs 4 vs 5 blocks of 4 warps per SM for the IPL=1 occupancy build
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/tp3.so build/ab/tp4.so build/ab/tp5.so
python - <<'PY'
import numpy as np
a=np.load('gpurun_out/c5ab_tp3.npy')
for n in ('tp4','tp5'):
    b=np.load('gpurun_out/c5ab_%s.npy' % n)
    same = all((a[f]==b[f]).all() for f in ('status','n_events','decision_hash','n_ok','n_completed')) and (a['attainment'].view('u8')==b['attainment'].view('u8')).all()
    print(n, 'bit-identical' if same else 'DIFFERENT')
PY
for W in c3; do for L in tp3 tp4 tp5; do ARROW_SIM_LIB=build/ab/$L.so python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W $L %.1f ms' % d['ms_per_step'])"; done; done
