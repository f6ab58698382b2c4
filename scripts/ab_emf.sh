set -u
for i in 1 2; do for F in 3 4 6 8; do
ARROW_EM_FACTOR=$F ARROW_C5_SAMPLE=16384 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 F=$F %.1f ms' % d['ms_per_step'])"
done; done
for F in 3 4 6; do
ARROW_EM_FACTOR=$F python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 F=$F %.1f ms' % d['ms_per_step'])"
done
