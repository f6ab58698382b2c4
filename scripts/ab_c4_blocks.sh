for i in 1 2 3; do for L in build/ab/cur.so build/ab/ipl2b2.so; do n=$(basename $L .so)
ARROW_SIM_LIB=$L python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $n %.1f ms' % d['ms_per_step'])"
done; done
