set -u
OUT=gpurun_out; TAG=r2e
make -s -j8 lib oracle emu > $OUT/build_$TAG.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build_$TAG.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest gpu rc=$?"; tail -3 $OUT/pytest_gpu_$TAG.log
timeout 300 python __graft_entry__.py > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke_$TAG.log
# compute-sanitizer (memcheck, racecheck) on the golden suite subset, both builds
cat > /tmp/san.py <<'PY'
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import harness as H
from paper_2505_11916_b200._backend import CudaEvaluator
idx = [m for m in H.golden_index() if not (m["error"] and m["error"][0] == "ValueError") and not m["name"].startswith(("c2_", "c3_", "c4_", "c5_"))]
items = [(m, H.golden_arrays(m)) for m in idx if m["stall_limit"] == 500000][:16]
for build in ("latency", "throughput"):
    for audit in (False, True):
        ev = CudaEvaluator(build=build, audit=audit)
        cb = H.compile_golden(items)
        hb = ev.execute(cb, H.spec_for(items))
        for s, (m, a) in enumerate(items):
            H.check_vs_golden(m, a, hb, s)
print("sanitized runs ok")
PY
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python /tmp/san.py > $OUT/sanitizer_memcheck_$TAG.log 2>&1; echo "memcheck rc=$?"; tail -3 $OUT/sanitizer_memcheck_$TAG.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python /tmp/san.py > $OUT/sanitizer_racecheck_$TAG.log 2>&1; echo "racecheck rc=$?"; tail -3 $OUT/sanitizer_racecheck_$TAG.log
