"""ctypes binding of libevb.so (the C ABI declared in include/evb.h).

The shared library is built in-tree (paper_2505_17430_b200/libevb.so) by
``__graft_entry__.build()``.  There is no fallback: if the library is missing or fails to load,
importing this module raises, and every compute entry point either launches the sm_100a kernels
or raises the mapped reference exception type.
"""
from __future__ import annotations

import ctypes
import os
import re
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
LIB_PATH = PKG_DIR / "libevb.so"
HEADER_PATH = PKG_DIR.parent / "include" / "evb.h"

EVB_OK = 0
EVB_ERR_INVALID_ARGUMENT = 1
EVB_ERR_CONFIG = 2
EVB_ERR_LOGIC = 3
EVB_ERR_RUNTIME = 4

EVB_F32 = 0
EVB_F64 = 1


class EvbError(RuntimeError):
    """Base of the mapped error types."""


class ConfigError(EvbError):
    """evobench::config_error (common.hpp:12-15)."""


class InvalidArgument(EvbError, ValueError):
    """std::invalid_argument (problems/batch.hpp:250-252)."""


class LogicError(EvbError):
    """std::logic_error (de/engine.hpp:32-33)."""


class DeviceError(EvbError):
    """std::runtime_error: CUDA / allocation failures."""


_ERRORS = {
    EVB_ERR_INVALID_ARGUMENT: InvalidArgument,
    EVB_ERR_CONFIG: ConfigError,
    EVB_ERR_LOGIC: LogicError,
    EVB_ERR_RUNTIME: DeviceError,
}

_lib = None


def declared_symbols() -> list[str]:
    """Every function the C header declares (used by the ABI test)."""
    text = HEADER_PATH.read_text()
    return sorted(set(re.findall(r"EVB_API\s+[\w\s\*]+?\b(evb_\w+)\s*\(", text)))


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)"
        )
    L = ctypes.CDLL(str(LIB_PATH), mode=os.RTLD_LAZY | ctypes.RTLD_GLOBAL)
    c_int, c_double, c_void_p, c_int64 = ctypes.c_int, ctypes.c_double, ctypes.c_void_p, ctypes.c_int64
    P = ctypes.POINTER
    sig = {
        "evb_abi_version": (c_int, []),
        "evb_last_error": (ctypes.c_char_p, []),
        "evb_device_info": (c_int, [c_int, P(c_int), P(c_int), P(c_int), P(c_int), P(c_int)]),
        "evb_problem_create_base": (c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_double, P(c_void_p)]),
        "evb_problem_create_hybrid": (
            c_int,
            [c_int, c_int, c_void_p, c_void_p, c_double, c_int, c_void_p, c_void_p, c_void_p, P(c_void_p)],
        ),
        "evb_problem_create_composition": (
            c_int,
            [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double, P(c_void_p)],
        ),
        "evb_problem_destroy": (c_int, [c_void_p]),
        "evb_problem_dim": (c_int, [c_void_p]),
        "evb_problem_dtype": (c_int, [c_void_p]),
        "evb_scratch_create": (c_int, [P(c_void_p)]),
        "evb_scratch_destroy": (c_int, [c_void_p]),
        "evb_evaluate_batch": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
        "evb_evaluate_batch_multi": (
            c_int,
            [c_void_p, c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_int64, c_void_p],
        ),
        "evb_evaluate_batch_host": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p]),
        "evb_evaluate_batch_host_many": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int64, c_int64, c_void_p]),
        "evb_evaluate_batch_problems": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                                c_void_p]),
        "evb_launch_count": (c_int, []),
        "evb_probe_peak_tflops": (c_int, [c_int, c_int, P(c_double)]),
        "evb_probe_umma_tf32_tflops": (c_int, [c_int, P(c_double)]),
        "evb_probe_umma_f16_tflops": (c_int, [c_int, P(c_double)]),
        "evb_scratch_host_staging": (c_int, [c_void_p, ctypes.c_size_t, P(c_void_p)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    _register_extra(L)
    return L


_extra_sigs: list = []


def register_signatures(sigs: dict) -> None:
    """Later modules (de, pso, runs, rng) add their entry points here."""
    _extra_sigs.append(sigs)
    if _lib is not None:
        _apply(_lib, sigs)


def _apply(L, sigs):
    for name, (res, args) in sigs.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def _register_extra(L):
    for s in _extra_sigs:
        _apply(L, s)


def check(status: int, what: str = "") -> None:
    if status == EVB_OK:
        return
    msg = lib().evb_last_error().decode(errors="replace")
    raise _ERRORS.get(status, EvbError)(f"{what}: {msg}" if what else msg)


def launch_count() -> int:
    return int(lib().evb_launch_count())


def probe_peak_tflops(which: int = 0, iters: int = 20000) -> float:
    """Measured FP64 DMMA (which=0) or FP32 FFMA (which=1) throughput of this GPU, TFLOP/s."""
    v = ctypes.c_double()
    check(lib().evb_probe_peak_tflops(which, iters, ctypes.byref(v)), "evb_probe_peak_tflops")
    return float(v.value)


def probe_umma_f16_tflops(n: int = 256) -> float:
    """Measured dense tcgen05.mma kind::f16 throughput (M=128, N=n, K=16) of this GPU, TFLOP/s."""
    v = ctypes.c_double()
    check(lib().evb_probe_umma_f16_tflops(n, ctypes.byref(v)), "evb_probe_umma_f16_tflops")
    return float(v.value)


def probe_umma_tf32_tflops(n: int = 256) -> float:
    """Measured dense tcgen05.mma kind::tf32 throughput (M=128, N=n, K=8) of this GPU, TFLOP/s."""
    v = ctypes.c_double()
    check(lib().evb_probe_umma_tf32_tflops(n, ctypes.byref(v)), "evb_probe_umma_tf32_tflops")
    return float(v.value)
