#!/usr/bin/env bash
# Interleaved A/B of prebuilt libraries: C5 sample (bit-identity vs the first), then C3/C4/C2.
#   bash scripts/ab_many.sh build/ab/A.so build/ab/B.so [...]
set -u
ARROW_C5_SAMPLE=${ARROW_C5_SAMPLE:-16384} bash scripts/ab_c5.sh "$@"
python - "$@" <<'PY'
import sys, os, numpy as np
names = [os.path.basename(x)[:-3] for x in sys.argv[1:]]
a = np.load('gpurun_out/c5ab_%s.npy' % names[0])
for n in names[1:]:
    b = np.load('gpurun_out/c5ab_%s.npy' % n)
    same = all((a[f] == b[f]).all() for f in ('status', 'n_events', 'decision_hash', 'n_ok', 'n_completed', 'n_iterations')) \
        and all((a[f].view('u8') == b[f].view('u8')).all() for f in ('attainment', 'stall_time', 'p90_ttft', 'mean_tpot', 'span'))
    print(n, 'vs', names[0], 'bit-identical summaries' if same else 'DIFFERENT')
PY
for W in ${AB_WORKLOADS:-c3 c4 c2}; do for i in 1 2; do for L in "$@"; do n=$(basename $L .so)
ARROW_SIM_LIB=$L python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W $n %.1f ms' % d['ms_per_step'])"
done; done; done
