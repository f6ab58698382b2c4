set -u
# occupancy shape: 3x4 warps (tp3) vs 2x4 (8 warps/SM, 202 regs) vs 2-warp and 3-warp blocks at 168 regs
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/tp3.so build/ab/b2w4.so build/ab/b5w2.so build/ab/b3w3.so
for W in c3; do for L in tp3 b2w4 b5w2 b3w3; do ARROW_SIM_LIB=build/ab/$L.so python bench.py --workload $W --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W $L %.1f ms' % d['ms_per_step'])"; done; done
