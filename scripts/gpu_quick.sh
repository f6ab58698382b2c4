#!/usr/bin/env bash
# Quick GPU iteration: build, evaluator parity tests, C2 bench without the
# CPU baseline / components.  Usage: bash scripts/gpu_quick.sh [tag]
set -u
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
make -s lib > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_reference_behaviour.py -x -q > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_$TAG.log
ARROW_BENCH_DUMP=$OUT/summaries_$TAG.npy timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-components > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('ms_per_step %.2f value %.3e e2e %.3e' % (d['ms_per_step'], d['value'], d['e2e']['value']))"
