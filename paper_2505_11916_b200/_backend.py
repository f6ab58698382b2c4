"""ctypes binding of libarrow_sim.so and device buffer plumbing.

PyTorch is used only for device memory, streams and copies.  There is no
CPU fallback: without a CUDA device or without the built library every
entry point raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from . import _abi
from ._buffers import HostBuffers, OutputSpec
from ._compile import CompiledBatch

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libarrow_sim.so"
# RunConfig.audit=True: the same kernel built with -DARROW_AUDIT (per-step
# KV / partition checks, engine.py:279-282)
AUDIT_LIB_PATH = LIB_PATH.with_name("libarrow_sim_audit.so")

_libs: dict = {}


class EvaluatorUnavailable(RuntimeError):
    pass


def load_library(audit: bool = False) -> ctypes.CDLL:
    if audit not in _libs:
        path = AUDIT_LIB_PATH if audit else Path(os.environ.get("ARROW_SIM_LIB", LIB_PATH))
        if not path.exists():
            raise EvaluatorUnavailable(
                f"CUDA evaluator library not built: {path} (run `make lib` or __graft_entry__.build())"
            )
        lib = ctypes.CDLL(str(path))
        lib.arrow_sim_abi_version.restype = ctypes.c_int
        lib.arrow_sim_workspace_size.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t)]
        lib.arrow_sim_workspace_size.restype = ctypes.c_int
        lib.arrow_sim_run.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p]
        lib.arrow_sim_run.restype = ctypes.c_int
        lib.arrow_sim_slots.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
        lib.arrow_sim_slots.restype = ctypes.c_int
        lib.arrow_sim_status_string.argtypes = [ctypes.c_int]
        lib.arrow_sim_status_string.restype = ctypes.c_char_p
        if lib.arrow_sim_abi_version() != _abi.ABI_VERSION:
            raise EvaluatorUnavailable(f"{path.name} ABI version mismatch; rebuild")
        _libs[audit] = lib
    return _libs[audit]


_OUTPUT_FIELDS = (
    "summaries",
    "req_first",
    "req_last",
    "req_prefill",
    "req_decode",
    "req_decode_iter",
    "decisions",
    "snapshots",
    "iterlog",
    "diag",
)
_INPUT_FIELDS = ("order", "outmap")


class DeviceBatch:
    """Device mirror of a HostBuffers: inputs uploaded, outputs allocated.

    ``upload`` (host->device), ``launch`` and ``download`` (device->host) are
    separate so callers can time the kernel alone or the whole round trip.
    """

    def __init__(self, hb: HostBuffers, device) -> None:
        import torch

        self.torch = torch
        self.hb = hb
        self.device = device
        self.tensors: dict[str, object] = {}
        self.h2d_bytes = 0
        self.d2h_bytes = 0
        self._pinned: dict[str, object] = {}

    def _dev_empty(self, nbytes: int):
        return self.torch.empty(max(nbytes, 1), dtype=self.torch.uint8, device=self.device)

    def _stage(self, name: str, arr: np.ndarray):
        raw = np.ascontiguousarray(arr).view(np.uint8).reshape(-1)
        pin = self._pinned.get(name)
        if pin is None or pin.numel() < raw.size:
            pin = self.torch.empty(raw.size, dtype=self.torch.uint8, pin_memory=True)
            self._pinned[name] = pin
        pin.numpy()[: raw.size] = raw
        return pin[: raw.size]

    def upload(self, inputs=None) -> None:
        hb = self.hb
        cb = hb.cb
        src = {
            "arrival": cb.arrival,
            "input_len": cb.input_len,
            "output_len": cb.output_len,
            "scenarios": cb.scenarios,
            "order": hb.order,
            "outmap": hb.outmap,
        }
        if inputs:
            src.update(inputs)
        self.h2d_bytes = 0
        ds = cb.device_set
        if ds is not None:
            # generated traces are read in place (device_traces.py)
            if ds.device != self.device:
                raise ValueError(f"traces were generated on {ds.device}, the batch runs on {self.device}")
            for name in ("arrival", "input_len", "output_len"):
                src.pop(name)
                self.tensors[name] = getattr(ds, name)
        for name, arr in src.items():
            if arr is None:
                continue
            staged = self._stage(name, arr)
            t = self.tensors.get(name)
            if t is None or t.numel() < staged.numel():
                t = self._dev_empty(staged.numel())
                self.tensors[name] = t
            t[: staged.numel()].copy_(staged, non_blocking=True)
            self.h2d_bytes += staged.numel()
        for name in _OUTPUT_FIELDS:
            arr = getattr(hb, name)
            if arr is None or name in self.tensors:
                continue
            self.tensors[name] = self._dev_empty(arr.nbytes)

    def struct(self) -> _abi.Batch:
        b = _abi.Batch()
        self.hb.fill_sizes(b)
        for name in _abi.POINTER_FIELDS:
            t = self.tensors.get(name)
            setattr(b, name, None if t is None else t.data_ptr())
        return b

    def launch(self, evaluator: "CudaEvaluator", stream=None) -> None:
        evaluator.launch(self, stream)

    def download(self, fields=None) -> HostBuffers:
        hb = self.hb
        self.d2h_bytes = 0
        for name in fields or _OUTPUT_FIELDS:
            arr = getattr(hb, name)
            if arr is None:
                continue
            t = self.tensors[name]
            host = self.torch.from_numpy(arr.view(np.uint8).reshape(-1))
            host.copy_(t[: arr.nbytes])
            self.d2h_bytes += arr.nbytes
        return hb


class CudaEvaluator:
    """Owns the device, the library handle and a reusable workspace."""

    BUILDS = {None: 0, "latency": 1, "throughput": 2}  # ARROW_SIM_FORCE_* (include/arrow_sim.h)

    def __init__(self, device=None, build: str | None = None, audit: bool = False) -> None:
        """build: None picks the kernel build by batch size; "latency" /
        "throughput" force one (identical results, different speed).
        audit: the per-step checking build (RunConfig.audit)."""
        import torch

        self.flags = self.BUILDS[build]
        if not torch.cuda.is_available():
            raise EvaluatorUnavailable("no CUDA device: the Arrow evaluator runs only on the GPU (no CPU fallback)")
        self.torch = torch
        self.lib = load_library(audit)
        self.audit = audit
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self._ws = None

    def workspace_for(self, b: _abi.Batch):
        need = ctypes.c_size_t(0)
        with self.torch.cuda.device(self.device):
            rc = self.lib.arrow_sim_workspace_size(ctypes.addressof(b), ctypes.byref(need))
        if rc:
            raise RuntimeError(f"arrow_sim_workspace_size failed: cuda error {rc}")
        if self._ws is None or self._ws.numel() < need.value:
            self._ws = None
            self._ws = self.torch.empty(need.value, dtype=self.torch.uint8, device=self.device)
        return self._ws, need.value

    def slots(self, b: _abi.Batch) -> int:
        n = ctypes.c_int(0)
        with self.torch.cuda.device(self.device):
            rc = self.lib.arrow_sim_slots(ctypes.addressof(b), ctypes.byref(n))
        if rc:
            raise RuntimeError(f"arrow_sim_slots failed: cuda error {rc}")
        return n.value

    def launch(self, db: DeviceBatch, stream=None) -> None:
        b = db.struct()
        ws, nbytes = self.workspace_for(b)
        s = stream if stream is not None else self.torch.cuda.current_stream(self.device)
        with self.torch.cuda.device(self.device):
            rc = self.lib.arrow_sim_run(ctypes.addressof(b), ws.data_ptr(), nbytes, ctypes.c_void_p(s.cuda_stream))
        if rc:
            raise RuntimeError(f"arrow_sim_run failed: cuda error {rc}")

    def prepare(self, cb: CompiledBatch, spec: OutputSpec, order=None) -> DeviceBatch:
        hb = HostBuffers(cb, spec, order)
        hb.flags = self.flags
        db = DeviceBatch(hb, self.device)
        db.upload()
        return db

    def execute(self, cb: CompiledBatch, spec: OutputSpec, order=None) -> HostBuffers:
        db = self.prepare(cb, spec, order)
        self.launch(db)
        hb = db.download()
        self.torch.cuda.synchronize(self.device)
        return hb


_default: dict = {}


def default_evaluator(audit: bool = False) -> CudaEvaluator:
    import torch

    dev = torch.cuda.current_device() if torch.cuda.is_available() else None
    ev = _default.get((dev, audit))
    if ev is None:
        ev = CudaEvaluator(audit=audit)
        _default[(dev, audit)] = ev
    return ev
