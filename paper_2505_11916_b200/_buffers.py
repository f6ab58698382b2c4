"""Output placement and host-side buffers for one batch launch.

``OutputSpec`` says which optional outputs a launch produces; ``Layout``
computes every per-scenario offset (the ``arrow_outmap_t`` array);
``HostBuffers`` owns numpy arrays of the right dtypes.  The CUDA backend
mirrors these as device tensors; the test harness hands the host arrays
straight to the CPU oracle.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from ._compile import CompiledBatch


@dataclass
class OutputSpec:
    requests: bool = False
    decisions: bool = False
    snapshots: bool = False
    iterlog: bool = False
    diag: bool = False
    tokens: bool = False                # CPU oracle only
    decision_factor: float = 1.0        # capacity multipliers (grown on overflow)
    snapshot_factor: float = 1.0
    iterlog_factor: float = 1.0

    @property
    def any(self) -> bool:
        return self.requests or self.decisions or self.snapshots or self.iterlog or self.diag or self.tokens


def _req_counts(cb: CompiledBatch) -> np.ndarray:
    return cb.scenarios["n_requests"].astype(np.int64)


@dataclass
class Layout:
    outmap: np.ndarray | None
    n_req: int
    n_dec: int
    n_snap: int
    n_iter: int
    n_diag: int
    n_tok: int


def make_layout(cb: CompiledBatch, spec: OutputSpec) -> Layout:
    S = cb.n
    if not spec.any:
        return Layout(None, 0, 0, 0, 0, 0, 0)
    om = np.full(S, -1, dtype=_abi.OUTMAP_DTYPE)
    om["decision_capacity"] = 0
    om["snapshot_capacity"] = 0
    om["iterlog_stride"] = 0
    n = _req_counts(cb)
    N = cb.scenarios["n_instances"].astype(np.int64)
    req = dec = snap = it = diag = tok = 0
    for s in range(S):
        ns, Ns = int(n[s]), int(N[s])
        if spec.requests:
            om["req_offset"][s] = req
            req += ns
        if spec.decisions:
            cap = int((2 * ns + 64) * spec.decision_factor)
            om["decision_offset"][s] = dec
            om["decision_capacity"][s] = cap
            dec += cap
        if spec.snapshots:
            tr = cb.table.entries[cb.trace_index[s]]
            span = float(tr.arrival[-1] * cb.scenarios["arrival_scale"][s]) if ns else 0.0
            ticks = int((span / cb.scenarios["monitor_period"][s] + 64) * spec.snapshot_factor)
            cap = Ns * ticks
            om["snapshot_offset"][s] = snap
            om["snapshot_capacity"][s] = cap
            snap += cap
        if spec.iterlog:
            tr = cb.table.entries[cb.trace_index[s]]
            work = int(tr.output_len.astype(np.int64).sum() + tr.input_len.astype(np.int64).sum() // 64)
            stride = int((work + 1024) * spec.iterlog_factor)
            om["iterlog_offset"][s] = it
            om["iterlog_stride"][s] = stride
            it += stride * Ns
        if spec.diag:
            om["diag_offset"][s] = diag
            diag += Ns
        if spec.tokens:
            tr = cb.table.entries[cb.trace_index[s]]
            om["token_offset"][s] = tok
            tok += int(tr.output_len.astype(np.int64).sum())
    return Layout(om, req, dec, snap, it, diag, tok)


class HostBuffers:
    """numpy arrays for every input and requested output of a batch."""

    def __init__(self, cb: CompiledBatch, spec: OutputSpec, order: np.ndarray | None = None) -> None:
        self.cb = cb
        self.spec = spec
        self.flags = 0  # arrow_batch_t.flags (kernel build override, see arrow_sim.h)
        self.layout = lay = make_layout(cb, spec)
        self.order = None if order is None else np.ascontiguousarray(order, dtype=np.int32)
        self.summaries = np.zeros(cb.n, dtype=_abi.SUMMARY_DTYPE)
        self.outmap = lay.outmap
        one = lambda n, dt: np.zeros(max(n, 1), dtype=dt)  # noqa: E731
        self.req_first = one(lay.n_req, np.float64) if spec.requests else None
        self.req_last = one(lay.n_req, np.float64) if spec.requests else None
        self.req_prefill = one(lay.n_req, np.int32) if spec.requests else None
        self.req_decode = one(lay.n_req, np.int32) if spec.requests else None
        self.req_decode_iter = one(lay.n_req, np.int32) if spec.requests else None
        self.decisions = one(lay.n_dec, _abi.DECISION_DTYPE) if spec.decisions else None
        self.snapshots = one(lay.n_snap, _abi.SNAPSHOT_DTYPE) if spec.snapshots else None
        self.iterlog = one(lay.n_iter, np.float64) if spec.iterlog else None
        self.diag = one(lay.n_diag, _abi.INSTDIAG_DTYPE) if spec.diag else None
        self.token_times = one(lay.n_tok, np.float64) if spec.tokens else None

    def fill_sizes(self, b: _abi.Batch) -> None:
        z = self.cb.sizes
        b.n_scenarios = self.cb.n
        b.flags = self.flags
        b.max_requests = z["max_requests"]
        b.max_instances = z["max_instances"]
        b.queue_capacity = z["queue_capacity"]
        b.emission_capacity = z["emission_capacity"]
        b.running_capacity = z["running_capacity"]
        b.fifo_capacity = z["fifo_capacity"]

    def host_struct(self) -> _abi.Batch:
        """arrow_batch_t pointing at these host arrays (CPU oracle / emulator)."""
        b = _abi.Batch()
        self.fill_sizes(b)

        def ptr(a):
            return None if a is None else a.ctypes.data

        cb = self.cb
        b.arrival = ptr(cb.arrival)
        b.input_len = ptr(cb.input_len)
        b.output_len = ptr(cb.output_len)
        b.scenarios = ptr(cb.scenarios)
        b.order = ptr(self.order)
        b.outmap = ptr(self.outmap)
        b.summaries = ptr(self.summaries)
        b.req_first = ptr(self.req_first)
        b.req_last = ptr(self.req_last)
        b.req_prefill = ptr(self.req_prefill)
        b.req_decode = ptr(self.req_decode)
        b.req_decode_iter = ptr(self.req_decode_iter)
        b.decisions = ptr(self.decisions)
        b.snapshots = ptr(self.snapshots)
        b.iterlog = ptr(self.iterlog)
        b.diag = ptr(self.diag)
        b.token_times = ptr(self.token_times)
        return b

    # -- per-scenario views ------------------------------------------------

    def req_slice(self, s: int) -> slice:
        off = int(self.outmap["req_offset"][s])
        return slice(off, off + int(self.cb.scenarios["n_requests"][s]))

    def decisions_of(self, s: int) -> np.ndarray:
        off = int(self.outmap["decision_offset"][s])
        n = int(min(self.summaries["n_decisions"][s], self.outmap["decision_capacity"][s]))
        return self.decisions[off : off + n]

    def snapshots_of(self, s: int) -> np.ndarray:
        off = int(self.outmap["snapshot_offset"][s])
        n = int(min(self.summaries["n_snapshots"][s], self.outmap["snapshot_capacity"][s]))
        return self.snapshots[off : off + n]

    def iterlog_of(self, s: int, inst: int) -> np.ndarray:
        stride = int(self.outmap["iterlog_stride"][s])
        off = int(self.outmap["iterlog_offset"][s]) + inst * stride
        return self.iterlog[off : off + stride]

    def diag_of(self, s: int) -> np.ndarray:
        off = int(self.outmap["diag_offset"][s])
        return self.diag[off : off + int(self.cb.scenarios["n_instances"][s])]

    def tokens_of(self, s: int, rid: int) -> np.ndarray:
        tr = self.cb.table.entries[self.cb.trace_index[s]]
        starts = np.concatenate(([0], np.cumsum(tr.output_len.astype(np.int64))))
        off = int(self.outmap["token_offset"][s])
        return self.token_times[off + starts[rid] : off + starts[rid + 1]]
