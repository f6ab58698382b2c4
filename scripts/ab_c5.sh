#!/usr/bin/env bash
# A/B of prebuilt libraries on a seeded C5 sample (throughput build), interleaved:
#   ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/libA.so build/ab/libB.so [...]
export ARROW_C5_SAMPLE=${ARROW_C5_SAMPLE:-16384}
mkdir -p gpurun_out
for i in 1 2; do for L in "$@"; do
  n=$(basename $L .so)
  ARROW_SIM_LIB=$L ARROW_BENCH_DUMP=gpurun_out/c5ab_$n.npy python bench.py --workload c5 --steps 2 --warmup 1 \
    --no-cpu-baseline --no-components > gpurun_out/c5ab_$n.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c5ab_$n.json')); print('$n', '%.1f ms' % d['ms_per_step'], '%.3e req/s' % d['value'])"
done; done
