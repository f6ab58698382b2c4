#!/usr/bin/env bash
# A/B timing of the trace_stats scan across prebuilt libraries, interleaved:
#   bash scripts/ab_stats.sh build/ab/libA.so build/ab/libB.so [...]
mkdir -p gpurun_out
for i in 1 2; do for L in "$@"; do
  n=$(basename $L .so)
  ARROW_SIM_LIB=$L python scripts/bench_stats.py --cpu-sample 1000 > gpurun_out/abs_$n.json 2> gpurun_out/abs_$n.err
  python -c "import json; d=json.loads(open('gpurun_out/abs_$n.json').read().strip().splitlines()[-1]); print('$n', '%.4f ms' % d['ms_per_scan'], 'frac %.4f' % d['roofline']['frac'])" || tail -3 gpurun_out/abs_$n.err
done; done
