#!/usr/bin/env bash
# Round-end style GPU run: build, all GPU tests, smoke, default bench (C5) +
# reference arm, C2-C4 bench lines, ncu capture of C4 (two instances per lane).
set -u
OUT=gpurun_out; TAG=${1:-final}
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi_$TAG.txt 2>&1
make -s -j8 lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -2 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
ARROW_BENCH_DUMP=$OUT/c5sum_$TAG.npy timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('C5 ms %.1f value %.4g e2e %.4g cpu %.4g clocks %s' % (d['ms_per_step'], d['value'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value', 0), d['clocks']))"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
for W in c4 c3 c2; do
timeout 900 python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline --no-components > $OUT/bench_${W}_$TAG.json 2> $OUT/bench_${W}_$TAG.err; echo "bench $W rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_${W}_$TAG.json')); print('$W ms %.1f value %.4g e2e %.4g' % (d['ms_per_step'], d['value'], d['e2e']['value']))"
done
if [ "${NCU_C4:-0}" = "1" ]; then
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_c4_$TAG -f \
  python bench.py --workload c4 --steps 1 --warmup 0 --no-cpu-baseline --no-components > $OUT/ncu_c4_$TAG.log 2>&1; echo "ncu c4 rc=$?"
fi
