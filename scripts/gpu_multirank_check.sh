# N>1 bench code path on a single GPU (two ranks sharing cuda:0, gloo backend):
# cost-balanced split, device gather, assembly, e2e gather.  Not a scaling
# measurement (both ranks share one GPU).
set -u
make -s lib >/dev/null 2>&1
ARROW_BENCH_BACKEND=gloo ARROW_C5_SAMPLE=2048 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 1 --warmup 1 --no-cpu-baseline --no-components \
  > gpurun_out/multirank.json 2> gpurun_out/multirank.err; echo "rc=$?"; tail -3 gpurun_out/multirank.err
python -c "import json; d=json.load(open('gpurun_out/multirank.json')); print(d['n_gpus'], d['config']['status_counts'], d['config']['scenarios'], d['value'])"
ARROW_C5_SAMPLE=2048 ARROW_BENCH_DUMP=gpurun_out/one.npy python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-components > /dev/null 2>&1
