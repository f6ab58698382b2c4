set -u
make -s -j8 lib oracle emu > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_probe2.log 2>&1; echo "pytest gpu rc=$?"; tail -1 gpurun_out/pytest_gpu_probe2.log
for i in 1 2 3; do for L in build/ab/r2x.so build/ab/probe2.so; do n=$(basename $L .so)
ARROW_SIM_LIB=$L ARROW_BENCH_DUMP=gpurun_out/c4_$n.npy python bench.py --workload c4 --steps 3 --warmup 1 --no-cpu-baseline --no-components 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4 $n %.1f ms' % d['ms_per_step'])"
done; done
python -c "
import numpy as np
a=np.load('gpurun_out/c4_r2x.npy'); b=np.load('gpurun_out/c4_probe2.npy')
f=[x for x in a.dtype.names if x not in ('cycles','reserved')]
print('c4 differing:', [x for x in f if not (np.ascontiguousarray(a[x]).view('u1')==np.ascontiguousarray(b[x]).view('u1')).all()])"
