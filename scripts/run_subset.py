"""Launch a subset of a named workload once (for ncu captures of one scenario class).
    python scripts/run_subset.py c2 27,28,29,30
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2505_11916_b200 import engine, workloads as W  # noqa: E402
from paper_2505_11916_b200._backend import CudaEvaluator  # noqa: E402
from paper_2505_11916_b200._buffers import OutputSpec  # noqa: E402
from paper_2505_11916_b200._compile import compile_batch  # noqa: E402

name, ids = sys.argv[1], [int(x) for x in sys.argv[2].split(",")]
scs = getattr(W, name)()
cb = compile_batch([scs[i] for i in ids], engine.STALL_EVENT_LIMIT)
ev = CudaEvaluator()
db = ev.prepare(cb, OutputSpec())
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 1):
    ev.launch(db)
hb = db.download(["summaries"])
torch.cuda.synchronize()
for i, r in zip(ids, hb.summaries):
    print(i, scs[i].label, int(r["status"]), int(r["n_events"]), int(r["cycles"]), int(r["n_serial_steps"]), int(r["n_parallel_steps"]))
