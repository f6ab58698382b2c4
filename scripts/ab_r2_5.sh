set -u
ROUNDS=2 bash scripts/ab.sh build/ab/cur.so build/ab/e1.so build/ab/lat1.so
ARROW_C5_SAMPLE=16384 bash scripts/ab_c5.sh build/ab/cur.so build/ab/e1.so
make -s -j8 lib oracle emu > gpurun_out/build_r2g.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2g.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/pytest_gpu_r2g.log
