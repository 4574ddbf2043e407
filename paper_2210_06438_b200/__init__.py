"""taskfuse-b200: B200-native strategy-3 work aggregation for the hydro
reconstruct+flux hot path of arXiv 2210.06438 (reference package `taskfuse`).

Sub-modules mirror the reference layout:
  errors         taskfuse/errors.py
  ops            tensor wrappers over the C ABI (include/taskfuse_b200.h)
  hydro          taskfuse/hydro (kernels, scenario, step)
  aggregator     taskfuse/aggregator.py (formation core in C++)
  bufferpool     taskfuse/bufferpool.py (pinned host + device)
  executorpool   taskfuse/executorpool.py (CUDA streams)
  device         the device seam of taskfuse/device.py on real CUDA
  sched          taskfuse/sched.py task API in real time
"""

from .errors import (CapacityError, DeadlockError, OrderingViolationError,
                     SimError, TaskfuseCudaError, UsageError, ValidationError)

__version__ = "0.1.0"

__all__ = ["CapacityError", "DeadlockError", "OrderingViolationError",
           "SimError", "TaskfuseCudaError", "UsageError", "ValidationError"]
