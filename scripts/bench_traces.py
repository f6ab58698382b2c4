"""Throughput of the device workload generator.

    python scripts/bench_traces.py [--seeds 8192] [--steps 5]

Generates the bundled bursty workload (traces.py:267-286, 2 606 requests per
seed) for --seeds seeds per launch; reports generated requests/s on the
device (CUDA events on the launch stream, after warm-up) next to the numpy
reference generator timed on a sample of seeds on one host core.  Prints
one JSON line.
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from dataclasses import replace
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def measure(seeds: int, steps: int = 5, warmup: int = 2, cpu_sample: int = 8) -> dict:
    args = argparse.Namespace(seeds=seeds, steps=steps, warmup=warmup, cpu_sample=cpu_sample)

    import ctypes

    import numpy as np
    import torch

    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200 import _abi, device_traces

    base = arrow.traces.SyntheticParams(
        duration_s=360.0, base_rate=4.0, input_log_mean=np.log(420.0), input_log_sigma=0.55,
        output_log_mean=np.log(130.0), output_log_sigma=0.5,
        bursts=(arrow.BurstEpisode(50.0, 25.0, 5.0), arrow.BurstEpisode(150.0, 30.0, 4.0),
                arrow.BurstEpisode(260.0, 25.0, 5.0)),
        max_input=3500, max_output=900, seed=0)
    params = [replace(base, seed=20240817 + s) for s in range(args.seeds)]
    ts = arrow.gen_synthetic_batch(params)          # sizes the buffers, checks status
    total = int(ts.counts.sum())
    lib = device_traces._load()
    specs = np.zeros(len(params), dtype=_abi.SYNTH_DTYPE)
    for i, p in enumerate(params):
        specs[i] = device_traces.synth_record(p, int(ts.offsets[i]), int(ts.counts[i]))
    d_specs = torch.from_numpy(specs.view(np.uint8).copy()).cuda()
    d_res = torch.empty(len(params) * _abi.SYNTH_RESULT_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def launch():
        rc = lib.arrow_synth_run(d_specs.data_ptr(), len(params), ts.arrival.data_ptr(), ts.input_len.data_ptr(),
                                 ts.output_len.data_ptr(), d_res.data_ptr(), ctypes.c_void_p(stream.cuda_stream))
        assert rc == 0, rc

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        launch()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    # bytes written per launch: 16 B per request + 64 B result per trace (+ specs read)
    bytes_per = total * 16 + len(params) * (_abi.SYNTH_RESULT_DTYPE.itemsize + _abi.SYNTH_DTYPE.itemsize)

    t0 = time.perf_counter()
    n_cpu = 0
    for p in params[: args.cpu_sample]:
        n_cpu += len(arrow.gen_synthetic(p))
    cpu_s = time.perf_counter() - t0
    return {
        "metric": "generated requests/s",
        "value": total / (ms / 1e3),
        "unit": "requests/s",
        "ms_per_launch": ms,
        "traces": len(params),
        "requests": total,
        "achieved_GBps": bytes_per / (ms * 1e6),
        "cpu_reference": {"value": n_cpu / cpu_s, "unit": "requests/s", "cores": 1,
                          "sample": f"{args.cpu_sample} seeds, numpy host generator (the reference's algorithm)"},
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--cpu-sample", type=int, default=8)
    a = ap.parse_args()
    print(json.dumps(measure(a.seeds, a.steps, a.warmup, a.cpu_sample)))


if __name__ == "__main__":
    main()
