#!/usr/bin/env bash
# Interleaved C2 (latency build) A/B of prebuilt libraries: bash scripts/ab_c2.sh A.so B.so ...
set -u
for i in 1 2 3; do for L in "$@"; do n=$(basename $L .so)
ARROW_SIM_LIB=$L python bench.py --workload c2 --steps 5 --warmup 2 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 $n %.2f ms' % d['ms_per_step'])"
done; done
