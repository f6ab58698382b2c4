"""Throughput of the trace_stats scan.

    python scripts/bench_stats.py [--requests 200000000] [--steps 10]

A sorted synthetic trace of --requests requests (arrival f64 + input i32 +
output i32 = 16 B/request, resident in HBM) is scanned --steps times; the
kernel is timed with CUDA events on its stream after warm-up, with a
256 MiB L2 flush between launches.  Reports requests/s, achieved GB/s on
the algorithmic 16 B/request and the fraction of MEASURED_PEAKS.json's HBM
bandwidth, next to the reference's trace_stats (CPU restatement) timed on a
--cpu-sample slice on one host core.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))


def hbm_peak() -> tuple[float, str]:
    try:
        d = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        for k in ("hbm_gbps_burst", "hbm_copy_gbps", "hbm_gbps"):
            if k in d:
                return float(d[k]), f"measured ({k})"
        for k, v in d.items():
            if "hbm" in k.lower() and isinstance(v, (int, float)):
                return float(v), f"measured ({k})"
    except Exception:
        pass
    return 6547.5, "fallback"


def measure(requests: int, steps: int = 10, warmup: int = 3, bucket: float = 60.0, cpu_sample: int = 200_000) -> dict:
    args = argparse.Namespace(requests=requests, steps=steps, warmup=warmup, bucket=bucket, cpu_sample=cpu_sample)
    import numpy as np
    import torch

    from paper_2505_11916_b200 import stats as ST

    n = args.requests
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    arrival = torch.cumsum(torch.rand(n, device=dev, dtype=torch.float64, generator=g) * 0.02, 0)
    inp = torch.randint(1, 8000, (n,), device=dev, dtype=torch.int32, generator=g)
    out = torch.randint(1, 2000, (n,), device=dev, dtype=torch.int32, generator=g)
    first, last = float(arrival[0]), float(arrival[-1])
    lo, hi = int(first // args.bucket), int(last // args.bucket)
    nb = hi - lo + 1
    lib = ST._lib()
    grid = ctypes.c_int32(0)
    lib.arrow_stats_grid(n, ctypes.byref(grid))
    bk = torch.empty((3, nb), dtype=torch.int64, device=dev)
    hist = torch.empty((2, ST.HIST_BINS), dtype=torch.int32, device=dev)
    parts = torch.empty(grid.value * ST.PARTIAL_DTYPE.itemsize, dtype=torch.uint8, device=dev)
    a = ST.StatsArgs(arrival.data_ptr(), inp.data_ptr(), out.data_ptr(), n, args.bucket, lo, nb, bk[0].data_ptr(),
                     bk[1].data_ptr(), bk[2].data_ptr(), hist[0].data_ptr(), hist[1].data_ptr(), parts.data_ptr(),
                     grid.value, 0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def launch():
        rc = lib.arrow_stats_run(ctypes.addressof(a), ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, rc

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    p = np.frombuffer(parts.cpu().numpy().tobytes(), dtype=ST.PARTIAL_DTYPE)
    assert int(p["count"].sum()) == n and int(p["out_of_window"].sum()) == 0
    gbps = 16.0 * n / (ms * 1e6)
    peak, src = hbm_peak()

    import stats_oracle as SO

    k = min(args.cpu_sample, n)
    sa, si, so = arrival[:k].cpu().numpy(), inp[:k].cpu().numpy(), out[:k].cpu().numpy()
    t0 = time.perf_counter()
    SO.trace_stats_arrays(sa, si, so, args.bucket)
    cpu_s = time.perf_counter() - t0
    return {
        "metric": "trace_stats requests/s", "value": n / (ms * 1e-3), "unit": "requests/s", "ms_per_scan": ms,
        "requests": n, "buckets": nb, "grid": grid.value,
        "roofline": {"bound": "hbm", "achieved": gbps, "peak": peak, "unit": "GB/s", "frac": gbps / peak,
                     "peak_source": src, "algorithmic_bytes_per_request": 16},
        "cpu_reference": {"value": k / cpu_s, "unit": "requests/s", "cores": 1,
                          "sample": f"first {k} requests, CPU restatement of traces.py:202-250"},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=200_000_000)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--bucket", type=float, default=60.0)
    ap.add_argument("--cpu-sample", type=int, default=200_000)
    a = ap.parse_args()
    print(json.dumps(measure(a.requests, a.steps, a.warmup, a.bucket, a.cpu_sample)))


if __name__ == "__main__":
    main()
