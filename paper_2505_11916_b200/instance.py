"""InstanceConfig (instance.py:33-51 of the reference).  The Instance state
machine itself lives in the CUDA evaluator (csrc/sim_core.cuh)."""

from .config import InstanceConfig

__all__ = ["InstanceConfig"]
