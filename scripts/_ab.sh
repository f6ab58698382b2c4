# A/B of the working tree (F, Python + lib) against D: the emission ring size is host-side
for i in 1 2 3; do for L in D F; do
  if [ $L = D ]; then export ARROW_EMCAP_X1=1; else unset ARROW_EMCAP_X1; fi
  ARROW_SIM_LIB=build/ab/lib$L.so ARROW_BENCH_DUMP=gpurun_out/sum_$L$i.npy python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-components > gpurun_out/c2_$L$i.json 2>/dev/null
  python -c "import json,numpy as np; b=json.load(open('gpurun_out/c2_$L$i.json')); s=np.load('gpurun_out/sum_$L$i.npy'); print('$L c2 ms %.2f max-scenario %d' % (b['ms_per_step'], int(np.argmax(s['cycles']))))"
done; done
for L in D F; do
  if [ $L = D ]; then export ARROW_EMCAP_X1=1; else unset ARROW_EMCAP_X1; fi
  ARROW_SIM_LIB=build/ab/lib$L.so ARROW_C5_SAMPLE=4096 python bench.py --workload c5 --steps 2 --warmup 1 --no-cpu-baseline --no-components > gpurun_out/c5_$L.json 2>/dev/null
  python -c "import json; b=json.load(open('gpurun_out/c5_$L.json')); print('$L c5 ms %.2f' % (b['ms_per_step']))"
done
