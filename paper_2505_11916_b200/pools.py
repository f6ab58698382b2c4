"""The pool state machine's legal edges (pools.py:20-31 of the reference);
membership and flips are maintained on the device (csrc/sim_core.cuh)."""

from .core import PoolKind

LEGAL_EDGES = frozenset(
    {
        (PoolKind.PREFILL, PoolKind.P_TO_D),
        (PoolKind.PREFILL, PoolKind.DECODE),
        (PoolKind.P_TO_D, PoolKind.DECODE),
        (PoolKind.P_TO_D, PoolKind.PREFILL),
        (PoolKind.DECODE, PoolKind.D_TO_P),
        (PoolKind.DECODE, PoolKind.PREFILL),
        (PoolKind.D_TO_P, PoolKind.PREFILL),
        (PoolKind.D_TO_P, PoolKind.DECODE),
    }
)
