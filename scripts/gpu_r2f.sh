set -u
OUT=gpurun_out; TAG=${1:-r2f}
make -s -j8 lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
ARROW_BENCH_DUMP=$OUT/c5sum_$TAG.npy timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"; tail -2 $OUT/bench_$TAG.err
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('C5 ms %.1f value %.4g e2e %.4g cpu %.4g clocks %s' % (d['ms_per_step'], d['value'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value', 0), d['clocks']))"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
for W in c4 c3 c2; do
timeout 900 python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline --no-components > $OUT/bench_${W}_$TAG.json 2> $OUT/bench_${W}_$TAG.err; echo "bench $W rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_${W}_$TAG.json')); print('$W ms %.1f value %.4g e2e %.4g' % (d['ms_per_step'], d['value'], d['e2e']['value']))"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-components > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
