"""B200-native (sm_100a) hot path of SEvoBench: batched shifted-rotated objective evaluation and
DE / PSO per-generation updates, behind the reference's module interfaces.

The compute lives in ``libevb.so`` (hand-written CUDA for sm_100a, C ABI in ``include/evb.h``);
this package is the host-side mirror of the reference interface over that ABI.
"""
from ._lib import (EVB_F32, EVB_F64, ConfigError, DeviceError, EvbError, InvalidArgument, LogicError,
                   launch_count)
from .problems import (BaseKind, EvalScratch, ProblemInstance, batched_evaluate, batched_evaluate_many,
                       evaluate_batch, evaluate_batch_multi, evaluate_batch_problems)

__all__ = [
    "EVB_F32", "EVB_F64", "ConfigError", "DeviceError", "EvbError", "InvalidArgument", "LogicError",
    "launch_count", "batched_evaluate_many", "evaluate_batch_problems", "BaseKind", "EvalScratch", "ProblemInstance", "batched_evaluate", "evaluate_batch",
    "evaluate_batch_multi",
]
