for i in 1 2 3; do for L in D F; do
  ARROW_SIM_LIB=build/ab/lib$L.so ARROW_BENCH_DUMP=gpurun_out/sum_$L$i.npy python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-components > gpurun_out/c2_$L$i.json 2>/dev/null
  python -c "import json,numpy as np; b=json.load(open('gpurun_out/c2_$L$i.json')); s=np.load('gpurun_out/sum_$L$i.npy'); c=s['cycles']; o=np.argsort(-c)[:3]; print('$L c2 ms %.2f top' % b['ms_per_step'], [(int(k), round(c[k]/1e6,1)) for k in o])"
done; done
for L in D F; do
  ARROW_SIM_LIB=build/ab/lib$L.so ARROW_C5_SAMPLE=4096 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline --no-components > gpurun_out/c5_$L.json 2>/dev/null
  python -c "import json; b=json.load(open('gpurun_out/c5_$L.json')); print('$L c5 ms %.2f' % (b['ms_per_step']))"
done
