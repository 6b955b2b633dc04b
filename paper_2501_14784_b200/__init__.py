"""B200-native DeServe stage-step path (arXiv 2501.14784) behind the pipesim interfaces.

Layout: ``csrc/cuda`` — sm_100a kernels and the ds_stage runtime; ``csrc/host`` — planner,
scheduler and executor (C++); ``include/deserve.h`` — the C ABI; this package — the Python
mirror of the reference's plan/run interface (``pipeline``) used by tests and bench.py.
"""
from ._native import (ConfigError, DsError, NoDeviceError, PlanError, SimError, check, lib,
                      n_devices)

__all__ = ["ConfigError", "DsError", "NoDeviceError", "PlanError", "SimError", "check", "lib",
           "n_devices"]
