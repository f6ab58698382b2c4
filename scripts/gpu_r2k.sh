set -u
OUT=gpurun_out; TAG=r2k
make -s -j8 lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; exit 1; }
ARROW_BENCH_DUMP=$OUT/c5sum_$TAG.npy timeout 1200 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('$OUT/bench_$TAG.json')); print('C5 ms %.1f value %.4g e2e %.4g cpu %.4g clocks %s' % (d['ms_per_step'], d['value'], d['e2e']['value'], (d['cpu_baseline'] or {}).get('value', 0), d['clocks']))"
ARROW_C5_SAMPLE=4096 timeout 900 ncu --set full --clock-control none --import-source on -k regex:arrow_sim_kernel -c 1 -o $OUT/prof_c5_$TAG -f \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-components > $OUT/ncu_c5_$TAG.log 2>&1; echo "ncu rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_$TAG.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-components > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
