"""Reference-written output files (TEST INFRASTRUCTURE; build container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/gen_golden_outputs.py

Runs three golden scenarios through the REAL reference (pdsim, imported
read-only from /root/reference/pkg/src) and stores the files its
``write_outputs`` writes (requests.csv, summary.json, monitor.csv,
decisions.jsonl; report.py:217-238), plus the ``pdsim compare`` summary CSV
(cli.py:26, 96-117) of a small strategies x rates grid, under
tests/golden/outputs/.  tests/test_outputs.py checks that this repo's
writers reproduce them byte for byte from the evaluator's results.
"""

from __future__ import annotations

import json
import shutil
import sys
import tempfile
from pathlib import Path

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))

import pdsim  # noqa: E402
import pdsim.cli as cli  # noqa: E402
import scenarios as S  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden" / "outputs"
NAMES = ("c1_rate4", "conservation_slo", "overload_flips")
COMPARE = dict(rates=["4", "8", "12"], strategies=["slo-aware", "minimal-load", "round-robin"])


def main() -> None:
    if OUT.exists():
        shutil.rmtree(OUT)
    OUT.mkdir(parents=True)
    index = json.loads((OUT.parent / "index.json").read_text())["scenarios"]
    metas = {m["name"]: m for m in index}
    for name in NAMES:
        m = metas[name]
        sc = next(s for s in S.catalogue(pdsim.TraceRequest) if s["name"] == name)
        config = pdsim.config_from_values(sc["values"])
        trace = pdsim.scale_trace(sc["trace"], sc["scale"]) if sc["scale"] != 1.0 else sc["trace"]
        result = pdsim.run(trace, config)
        pdsim.write_outputs(result, config.slo, OUT / name, decisions=True)
        assert m["error"] is None
    # pdsim compare on a 400-request slice of the bundled trace (config file
    # = the rate-sweep config of test_acceptance.py:55-72)
    trace = pdsim.bundled_bursty_trace()[:400]
    with tempfile.TemporaryDirectory() as tmp:
        tpath = Path(tmp) / "trace.csv"
        pdsim.save_trace(trace, tpath)
        cpath = OUT / "compare_config.txt"
        values = S.adaptive_vs_static(8, "slo-aware")
        cpath.write_text("".join(f"{k} = {v}\n" for k, v in values.items()))
        shutil.copy(tpath, OUT / "compare_trace.csv")
        rc = cli.main(["compare", str(tpath), "--config", str(cpath), "--rates", *COMPARE["rates"],
                       "--strategies", *COMPARE["strategies"], "--out", str(OUT / "compare.csv")])
        assert rc == 0
    (OUT / "README").write_text(__doc__)
    print("wrote", sorted(p.relative_to(OUT).as_posix() for p in OUT.rglob("*") if p.is_file()))


if __name__ == "__main__":
    main()
