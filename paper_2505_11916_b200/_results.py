"""Turn raw evaluator outputs back into the reference's Python objects.

* statuses -> the reference's exceptions with its exact messages
  (SimulationStallError engine.py:283-287, 305-316; AssertionError 288-290;
  RuntimeError scheduler.py:193; ZeroDivisionError scheduler.py:322)
* per-request first/last times + per-instance iteration log -> RequestRecord
  with full token_times (core.py:105-129)
* decision stream -> GlobalScheduler.decisions dicts (scheduler.py:104-122)
  and PoolSet.transitions (pools.py:84)
* snapshot records -> MonitorSnapshot series (monitor.py:56-73)
"""

from __future__ import annotations

import math

import numpy as np

from . import _abi
from ._buffers import HostBuffers
from .core import POOL_BY_CODE, RequestRecord, SLOConfig
from .monitor import InstanceStats, MonitorSnapshot


class SimulationStallError(RuntimeError):
    """Raised when the event loop stops making progress (engine.py:35-36)."""


def _stall_message(hb: HostBuffers, s: int, when) -> str:
    summ = hb.summaries[s]
    sc = hb.cb.scenarios[s]
    lines = [f"simulation stalled at t={when!r}: {int(summ['n_completed'])}/{int(summ['n_requests'])} requests complete"]
    if hb.diag is not None:
        cap = int(sc["kv_capacity"])
        for i, d in enumerate(hb.diag_of(s)):
            busy = None if math.isnan(d["busy_until"]) else float(d["busy_until"])
            lines.append(
                f"  instance {i}: pool={_abi.POOL_NAMES[int(d['pool'])]} kv={int(d['kv_used'])}/{cap} "
                f"running={int(d['running'])} waiting={int(d['waiting'])} migrating={int(d['migrating'])} "
                f"busy_until={busy!r}"
            )
    return "\n".join(lines)


def raise_for_status(hb: HostBuffers, s: int) -> None:
    summ = hb.summaries[s]
    st = int(summ["status"])
    if st == _abi.OK:
        return
    if st == _abi.STALLED:
        raise SimulationStallError(_stall_message(hb, s, float(summ["stall_time"])))
    if st == _abi.INCOMPLETE:
        raise SimulationStallError(_stall_message(hb, s, None))
    if st == _abi.NOT_DRAINED:
        raise AssertionError("instance not drained at end of run")
    if st == _abi.NO_INSTANCE:
        raise RuntimeError("no instance available for prefill dispatch")
    if st == _abi.ZERO_DIVISION:
        raise ZeroDivisionError("division by zero")
    if st == _abi.AUDIT_FAILED:
        raise AssertionError("audit: instance KV accounting or pool partition inconsistent (engine.py:279-282)")
    if st == _abi.BUFFER_OVERFLOW:
        raise OverflowError(f"evaluator buffer too small: {_abi.OVERFLOW_NAMES[int(summ['overflow'])]}")
    raise RuntimeError(f"evaluator invariant violated (status {_abi.STATUS_NAMES[st]})")


def token_times(hb: HostBuffers, s: int) -> list[list[float]]:
    """Rebuild every request's emission times: the first token from the
    prefill, then one per iteration of its decode instance from admission
    (every running decode is in every batch, instance.py:187-191)."""
    sl = hb.req_slice(s)
    first = hb.req_first[sl]
    dec = hb.req_decode[sl]
    dit = hb.req_decode_iter[sl]
    tr = hb.cb.table.entries[hb.cb.trace_index[s]]
    out = tr.output_len
    logs: dict[int, np.ndarray] = {}
    result = []
    for r in range(len(first)):
        m = int(out[r])
        if m == 1:
            result.append([float(first[r])])
            continue
        inst = int(dec[r]) & 0xFFFF
        log = logs.get(inst)
        if log is None:
            log = logs[inst] = hb.iterlog_of(s, inst)
        k0 = int(dit[r])
        result.append([float(first[r])] + log[k0 : k0 + m - 1].tolist())
    return result


def records(hb: HostBuffers, s: int, arrival_scaled: np.ndarray, ids: np.ndarray, slo: SLOConfig) -> list[RequestRecord]:
    times = token_times(hb, s)
    return [
        RequestRecord.from_token_times(int(ids[r]), float(arrival_scaled[r]), times[r], slo) for r in range(len(times))
    ]


def decision_dicts(hb: HostBuffers, s: int, ids: np.ndarray) -> list[dict]:
    out = []
    for d in hb.decisions_of(s):
        kind = int(d["kind"])
        t = float(d["time"])
        inst = int(d["instance"])
        code = int(d["code"])
        if kind == _abi.DEC_FLIP:
            out.append(
                {
                    "time": t,
                    "kind": "flip",
                    "instance": inst,
                    "from": _abi.POOL_NAMES[(code >> 3) & 3],
                    "to": _abi.POOL_NAMES[(code >> 5) & 3],
                    "trigger": _abi.TRIGGER_NAMES[code & 7],
                }
            )
        else:
            out.append(
                {
                    "time": t,
                    "kind": _abi.DECISION_KIND_NAMES[kind],
                    "request_id": int(ids[int(d["request"])]),
                    "instance": inst,
                    "branch": _abi.BRANCH_NAMES[code],
                }
            )
    return out


def transitions(decisions: list[dict]):
    by_name = {k.value: k for k in POOL_BY_CODE}
    return [(d["instance"], by_name[d["from"]], by_name[d["to"]]) for d in decisions if d["kind"] == "flip"]


def snapshots(hb: HostBuffers, s: int) -> list[MonitorSnapshot]:
    recs = hb.snapshots_of(s)
    N = int(hb.cb.scenarios["n_instances"][s])
    out = []
    for k in range(0, len(recs), N):
        group = recs[k : k + N]
        stats = tuple(
            InstanceStats(
                instance_id=int(g["instance"]),
                pool=POOL_BY_CODE[int(g["pool"])],
                running_tokens=int(g["running_tokens"]),
                kv_used=int(g["kv_used"]),
                queue_len=int(g["queue_len"]),
                pred_delay=float(g["pred_delay"]),
                avg_interval=None if math.isnan(g["avg_interval"]) else float(g["avg_interval"]),
                prefill_count=int(g["prefill_count"]),
                decode_count=int(g["decode_count"]),
            )
            for g in group
        )
        out.append(MonitorSnapshot(time=float(group[0]["time"]), per_instance=stats))
    return out
