"""Python-reference timing sample (build container only; TEST/MEASUREMENT
INFRASTRUCTURE).

The reference (pure-Python pdsim) cannot travel to the GPU box, so its own
speed is measured here: oracle/gen_golden.py ran the 32 stratified C5
scenarios (and the C3/C4 fixtures) through the real ``pdsim`` and recorded
each run's wall time in tests/golden/index.json.  This script adds the C
port's single-thread time on the same scenarios (same container) and writes
profiles/python_reference_sample.json, which bench.py reports as
``cpu_baseline.python_sample`` next to the port measured on the box.

    python scripts/python_ref_sample.py
"""

from __future__ import annotations

import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import harness as H  # noqa: E402


def main() -> None:
    rows = []
    for prefix in ("c5_", "c3_", "c4_"):
        metas = [m for m in H.golden_index() if m["name"].startswith(prefix) and m["error"] is None]
        for m in metas:
            a = H.golden_arrays(m)
            cb = H.compile_golden([(m, a)])
            t0 = time.perf_counter()
            hb, secs, _ = H.run_oracle_timed(cb, threads=1)
            port = time.perf_counter() - t0
            s = hb.summaries[0]
            rows.append(dict(name=m["name"], config=prefix[:2], requests=int(len(a["arrival"])),
                             events=int(s["n_events"]), python_s=m["wall_s"], port_s=port))
    model = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    model = next((ln.split(":", 1)[1].strip() for ln in model.splitlines() if ln.startswith("Model name")), "?")
    out = {"measured_on": f"build container, 1 core of {model} (CPython "
                          f"{sys.version.split()[0]}); the GPU box has no copy of the reference",
           "reference": "pdsim.run (real reference, imported read-only) via oracle/gen_golden.py",
           "per_config": {}}
    for cfg in ("c5", "c3", "c4"):
        rs = [r for r in rows if r["config"] == cfg]
        if not rs:
            continue
        req = sum(r["requests"] for r in rs)
        py = sum(r["python_s"] for r in rs)
        po = sum(r["port_s"] for r in rs)
        out["per_config"][cfg] = {"scenarios": len(rs), "requests": req, "events": sum(r["events"] for r in rs),
                                  "python_s": py, "port_s": po, "python_req_per_s_per_core": req / py,
                                  "port_req_per_s_per_core": req / po, "python_over_port": py / po}
    # whole sweeps run through the real reference by oracle/gen_golden_digest.py
    # (7 worker processes on the 8-core build container, so per-scenario wall
    # times include some contention)
    out["whole_sweeps"] = {}
    for cfg, total in (("c3", 1920), ("c4", 1080), ("c5", None)):
        path = ROOT / "tests" / "golden" / f"digest_{cfg}.npz"
        if not path.exists():
            continue
        with np.load(path) as z:
            wall = z["wall_s"]
            ids = z["id"]
            st = z["status"]
        import paper_2505_11916_b200.workloads as W
        reqs = sum(len(sc.trace) for sc in getattr(W, cfg)(ids))
        out["whole_sweeps"][cfg] = {"scenarios": int(len(ids)), "of": total or 98304, "requests": int(reqs),
                                    "stalled": int((st == 1).sum()), "python_core_s": float(wall.sum()),
                                    "python_req_per_s_per_core": float(reqs / wall.sum())}
    out["scenarios"] = rows
    path = ROOT / "profiles" / "python_reference_sample.json"
    path.write_text(json.dumps(out, indent=1))
    print(json.dumps(out["per_config"], indent=1))


if __name__ == "__main__":
    main()
