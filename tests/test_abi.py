"""The C-ABI boundary: the device library loads, exports every entry point
include/arrow_sim.h declares, and its struct layout matches the Python
mirrors byte for byte (no CUDA calls; runs without a GPU)."""

from __future__ import annotations

import ctypes
import re

import numpy as np
import pytest

import harness as H
from paper_2505_11916_b200 import _abi

LIB = H.ROOT / "paper_2505_11916_b200" / "lib" / "libarrow_sim.so"
HEADER = H.ROOT / "include" / "arrow_sim.h"


@pytest.fixture(scope="module")
def lib():
    if not LIB.exists():
        H._build("lib")
    return ctypes.CDLL(str(LIB))


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(arrow_sim_\w+)\s*\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert {"arrow_sim_run", "arrow_sim_workspace_size", "arrow_sim_abi_version", "arrow_sim_layout"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name


def test_abi_version(lib):
    lib.arrow_sim_abi_version.restype = ctypes.c_int
    assert lib.arrow_sim_abi_version() == _abi.ABI_VERSION


def test_struct_layout_matches_python_mirrors(lib):
    out = (ctypes.c_int64 * 512)()
    lib.arrow_sim_layout.restype = ctypes.c_int
    n = lib.arrow_sim_layout(out, 512)
    vals = list(out[:n])
    sizes, offs = vals[:7], vals[7:]
    dtypes = [_abi.SCENARIO_DTYPE, _abi.OUTMAP_DTYPE, _abi.SUMMARY_DTYPE, _abi.DECISION_DTYPE,
              _abi.SNAPSHOT_DTYPE, _abi.INSTDIAG_DTYPE]
    assert sizes == [d.itemsize for d in dtypes] + [ctypes.sizeof(_abi.Batch)]
    expected = []
    for d in dtypes:
        expected += [d.fields[f][1] for f in d.names]
    expected += [getattr(_abi.Batch, f).offset for f, _ in _abi.Batch._fields_]
    assert offs == expected


def test_status_strings(lib):
    lib.arrow_sim_status_string.restype = ctypes.c_char_p
    lib.arrow_sim_status_string.argtypes = [ctypes.c_int]
    assert [lib.arrow_sim_status_string(i).decode() for i in range(len(_abi.STATUS_NAMES))] == list(_abi.STATUS_NAMES)


def test_library_is_sm100a():
    """The device code is built for sm_100a only (no PTX JIT fallback)."""
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(LIB)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout
    ptx = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-ptx", str(LIB)], capture_output=True, text=True)
    assert ptx.stdout.strip() == ""


def test_product_fails_loudly_without_gpu():
    """No CPU fallback: without a CUDA device the drop-in API raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200._backend import EvaluatorUnavailable

    trace = [arrow.TraceRequest(0, 0.0, 100, 4)]
    with pytest.raises(EvaluatorUnavailable):
        arrow.run(trace, arrow.default_run_config())


TRACES_HEADER = H.ROOT / "include" / "arrow_traces.h"


def test_traces_header_symbols_exported(lib):
    text = TRACES_HEADER.read_text()
    names = sorted(set(re.findall(r"^\s*int\s+(arrow_\w+)\s*\(", text, re.M)))
    assert names == ["arrow_stats_grid", "arrow_stats_hist", "arrow_stats_layout", "arrow_stats_run",
                     "arrow_synth_layout", "arrow_synth_run"]
    for name in names:
        assert hasattr(lib, name), name


def test_synth_layout_matches_python_mirrors(lib):
    out = (ctypes.c_int64 * 64)()
    lib.arrow_synth_layout.restype = ctypes.c_int
    n = lib.arrow_synth_layout(out, 64)
    vals = list(out[:n])
    dts = [_abi.SYNTH_DTYPE, _abi.SYNTH_RESULT_DTYPE]
    expected = [d.itemsize for d in dts]
    for d in dts:
        expected += [d.fields[f][1] for f in d.names]
    assert vals == expected
    text = TRACES_HEADER.read_text()
    assert f"#define ARROW_SYNTH_MAX_BURSTS {_abi.SYNTH_MAX_BURSTS}" in text
    assert f"#define ARROW_SYNTH_MAX_SEED_WORDS {_abi.SYNTH_MAX_SEED_WORDS}" in text


def test_generator_fails_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2505_11916_b200 as arrow
    from paper_2505_11916_b200._backend import EvaluatorUnavailable

    with pytest.raises(EvaluatorUnavailable):
        arrow.gen_synthetic_batch([arrow.SyntheticParams(10.0, 1.0, 5.0, 0.5, 4.0, 0.5)])


def test_stats_layout_matches_python_mirrors(lib):
    from paper_2505_11916_b200 import stats as ST

    out = (ctypes.c_int64 * 64)()
    lib.arrow_stats_layout.restype = ctypes.c_int
    n = lib.arrow_stats_layout(out, 64)
    vals = list(out[:n])
    expected = [ST.PARTIAL_DTYPE.itemsize, ctypes.sizeof(ST.StatsArgs)]
    expected += [ST.PARTIAL_DTYPE.fields[f][1] for f in ST.PARTIAL_DTYPE.names]
    expected += [getattr(ST.StatsArgs, f).offset for f, _ in ST.StatsArgs._fields_]
    assert vals == expected
    text = TRACES_HEADER.read_text()
    assert f"#define ARROW_STATS_HIST_BINS {ST.HIST_BINS}" in text
    for name in ("arrow_stats_grid", "arrow_stats_run", "arrow_stats_hist", "arrow_stats_layout"):
        assert hasattr(lib, name), name
