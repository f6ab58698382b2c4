"""Strategy / SchedulerConfig (scheduler.py:25-45 of the reference).  The
dispatch and flip rules run inside the CUDA evaluator (csrc/sim_core.cuh)."""

from .config import SchedulerConfig, Strategy

__all__ = ["SchedulerConfig", "Strategy"]
