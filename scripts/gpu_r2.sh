#!/usr/bin/env bash
# Round-2 GPU check: parity tests, smoke, default bench (C5) + reference arm,
# optional extra workloads.  Usage (under gpurun): bash scripts/gpu_r2.sh TAG [extra workloads...]
set -u
TAG=${1:-r2}; shift || true
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
make -s lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
fi
if [ "${SKIP_BENCH:-0}" != "1" ]; then
ARROW_BENCH_DUMP=$OUT/c5sum_$TAG.npy timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -2 $OUT/bench_$TAG.err
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('C5 ms %.1f value %.4g e2e %.4g cpu %.4g' % (d['ms_per_step'], d['value'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value', 0)))"
fi
if [ "${SKIP_REF:-0}" != "1" ]; then
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_ref_$TAG.json')); print('reference value %.4g' % d['value'])"
fi
for W in "$@"; do
timeout 900 python bench.py --workload $W --steps 2 --warmup 1 --no-cpu-baseline --no-components > $OUT/bench_${W}_$TAG.json 2> $OUT/bench_${W}_$TAG.err; echo "bench $W rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_${W}_$TAG.json')); print('$W ms %.1f value %.4g e2e %.4g' % (d['ms_per_step'], d['value'], d['e2e']['value']))"
done
