#!/usr/bin/env bash
# A/B timing of two prebuilt libraries on the same box, interleaved:
#   bash scripts/ab.sh build/ab/libA.so build/ab/libB.so [rounds]
A=$1; B=$2; R=${3:-3}
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for L in A B; do
    if [ $L = A ]; then LIB=$A; else LIB=$B; fi
    ARROW_SIM_LIB=$LIB ARROW_BENCH_DUMP=gpurun_out/ab_$L$i.npy python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-components > gpurun_out/ab_$L$i.json 2>/dev/null
    python -c "import json,numpy as np; d=json.load(open('gpurun_out/ab_$L$i.json')); s=np.load('gpurun_out/ab_$L$i.npy'); print('$L ms %.2f sumcyc %.3fG max %.1fM' % (d['ms_per_step'], s['cycles'].sum()/1e9, s['cycles'].max()/1e6))"
  done
done
