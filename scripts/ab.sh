#!/usr/bin/env bash
# A/B timing of prebuilt libraries on the same box, interleaved:
#   ROUNDS=3 bash scripts/ab.sh build/ab/libA.so build/ab/libB.so [more.so ...]
# Prints ms/step and the summed / critical scenario cycles per library;
# summaries land in gpurun_out/ab_<index><round>.npy for bitwise comparison.
R=${ROUNDS:-3}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  n=0
  for LIB in "$@"; do
    n=$((n + 1))
    ARROW_SIM_LIB=$LIB ARROW_BENCH_DUMP=gpurun_out/ab_$n$i.npy python bench.py --workload ${WORKLOAD:-c2} --steps 3 --warmup 3 --no-cpu-baseline --no-components > gpurun_out/ab_$n$i.json 2>/dev/null
    python -c "import json,numpy as np; d=json.load(open('gpurun_out/ab_$n$i.json')); s=np.load('gpurun_out/ab_$n$i.npy'); print('$n $(basename $LIB) ms %.2f sumcyc %.3fG max %.1fM' % (d['ms_per_step'], s['cycles'].sum()/1e9, s['cycles'].max()/1e6))"
  done
done
