"""Golden vectors for the device workload generator (TEST INFRASTRUCTURE).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_traces.py

Runs the REAL reference generator ``pdsim.gen_synthetic`` (traces.py:159-175,
imported read-only from /root/reference/pkg/src, present only in the build
container) on every parameter set of oracle/synth_catalogue.py and stores
the traces in tests/golden/synth_traces.npz (arrival bits, input, output per
entry, plus the Python exception for parameter sets that raise).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))

import pdsim  # noqa: E402
from synth_catalogue import catalogue  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "synth_traces.npz"


def main() -> None:
    arrays = {}
    meta = []
    for name, kw in catalogue():
        kw = dict(kw)
        kw["bursts"] = tuple(pdsim.BurstEpisode(*b) for b in kw.get("bursts", ()))
        try:
            trace = pdsim.gen_synthetic(pdsim.SyntheticParams(**kw))
            err = None
        except Exception as exc:  # recorded, compared by type and message
            trace, err = [], f"{type(exc).__name__}: {exc}"
        arrays[f"{name}__arrival"] = np.array([r.arrival for r in trace], dtype=np.float64)
        arrays[f"{name}__input"] = np.array([r.input_len for r in trace], dtype=np.int64)
        arrays[f"{name}__output"] = np.array([r.output_len for r in trace], dtype=np.int64)
        meta.append(dict(name=name, n=len(trace), error=err))
        print(f"{name:20s} n={len(trace):5d} err={err}")
    arrays["meta"] = np.array(json.dumps(dict(generator="oracle/gen_golden_traces.py", numpy=np.__version__,
                                              python=sys.version.split()[0], entries=meta)))
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
