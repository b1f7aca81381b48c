"""ctypes loader of the parity checker (TEST INFRASTRUCTURE ONLY).

* ``C``   -> oracle/_build/liboracle.so : the plain-C restatement of the reference (evb_oracle.c)
* ``REF`` -> oracle/_ref/libevbref_exact.so : the unmodified reference headers (ref_driver.cpp),
             reference Release flags; ``REF_FAST`` the -O3 -march build used for CPU timing.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this module.  The product path (paper_2505_17430_b200) never does.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
C_LIB = HERE / "_build" / "liboracle.so"
REF_DIR = HERE / "_ref"

_c = None
_ref = None
_ref_fast = None

u64, i64, c_int, c_double, c_float, vp = (ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_float, ctypes.c_void_p)


def ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


def C():
    global _c
    if _c is None:
        if not C_LIB.exists():
            raise ImportError(f"{C_LIB} missing: run `make -C oracle` (or __graft_entry__.build())")
        L = ctypes.CDLL(str(C_LIB))
        sig = {
            "orc_rng_size": (c_int, []),
            "orc_rng_init": (None, [vp, u64, u64]),
            "orc_rng_scripted": (None, [vp, vp, i64]),
            "orc_next_u64": (u64, [vp]),
            "orc_rng_words": (None, [u64, u64, i64, i64, vp]),
            "orc_uniform_int_word": (c_int, [u64, c_int]),
            "orc_philox_block": (None, [vp, vp, vp]),
            "orc_philox_word": (u64, [u64, u64, u64]),
            "orc_philox_words": (None, [u64, u64, u64, i64, vp]),
            "orc_random_rotation": (None, [vp, c_int, vp]),
            "orc_draw_shift": (None, [vp, c_int, c_double, c_double, vp]),
            "orc_make_shift_rotation": (None, [u64, u64, c_int, vp, vp]),
            "orc_init_population": (None, [vp, c_int, c_int, c_double, c_double, vp]),
            "orc_init_population_seed": (None, [u64, u64, c_int, c_int, c_double, c_double, vp]),
            "orc_fast_cos": (c_float, [c_float]),
            "orc_fast_sin": (c_float, [c_float]),
            "orc_eval_batch_f64": (None, [c_int, c_int, vp, vp, c_double, i64, vp, i64, vp]),
            "orc_eval_batch_f32": (None, [c_int, c_int, vp, vp, c_float, i64, vp, i64, vp]),
            "orc_eval_scalar_f64": (c_double, [c_int, c_int, vp, vp, c_double, vp]),
            "orc_eval_scalar_f32": (c_float, [c_int, c_int, vp, vp, c_float, vp]),
            "orc_base_value_f64": (c_double, [c_int, vp, c_int]),
            "orc_eval_hybrid_f64": (None, [c_int, vp, vp, c_double, c_int, vp, vp, vp, i64, vp, i64, vp]),
            "orc_eval_hybrid_f32": (None, [c_int, vp, vp, c_float, c_int, vp, vp, vp, i64, vp, i64, vp]),
            "orc_eval_composition_f64": (None, [c_int, c_int, vp, vp, vp, vp, vp, vp, c_double, i64, vp, i64, vp]),
            "orc_eval_composition_f32": (None, [c_int, c_int, vp, vp, vp, vp, vp, vp, c_float, i64, vp, i64, vp]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _register(L, _extra_c)
        _c = L
    return _c


_extra_c: list = []
_extra_ref: list = []


def _register(L, lst):
    for sig in lst:
        for name, (res, args) in sig.items():
            if hasattr(L, name):
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args


def register_c(sig):
    _extra_c.append(sig)
    if _c is not None:
        _register(_c, [sig])


def register_ref(sig):
    _extra_ref.append(sig)
    for L in (_ref, _ref_fast):
        if L is not None:
            _register(L, [sig])


REF_SIG = {
    "ref_rng_words": (None, [u64, u64, i64, i64, vp]),
    "ref_make_shift_rotation": (None, [u64, u64, c_int, vp, vp]),
    "ref_init_population": (None, [u64, u64, c_int, c_int, c_double, c_double, vp]),
    "ref_make_instance_f64": (c_int, [c_int, c_int, c_int, u64, vp, vp, vp, vp]),
    "ref_eval_batch_f64": (None, [c_int, c_int, vp, vp, c_double, i64, vp, i64, vp]),
    "ref_eval_batch_f32": (None, [c_int, c_int, vp, vp, c_double, i64, vp, i64, vp]),
    "ref_eval_scalar_f64": (c_double, [c_int, c_int, vp, vp, c_double, vp]),
    "ref_eval_hybrid_f64": (None, [c_int, vp, vp, c_double, c_int, vp, vp, vp, i64, vp, i64, vp]),
    "ref_eval_composition_f64": (None, [c_int, c_int, vp, vp, vp, vp, vp, vp, c_double, i64, vp, i64, vp]),
    "ref_batch_job_create": (vp, [c_int, c_int, c_int, vp, vp, c_double, i64, vp]),
    "ref_batch_job_run": (None, [vp, c_int, vp]),
    "ref_batch_job_destroy": (None, [vp]),
    "ref_hardware_threads": (c_int, []),
}


def _load_ref(path: Path):
    L = ctypes.CDLL(str(path))
    _register(L, [REF_SIG])
    _register(L, _extra_ref)
    return L


def ref_available() -> bool:
    return (REF_DIR / "libevbref_exact.so").exists()


def REF():
    """Reference built with its own Release flags (parity)."""
    global _ref
    if _ref is None:
        p = REF_DIR / "libevbref_exact.so"
        if not p.exists():
            raise ImportError(f"{p} missing: run `make -C oracle ref` where /root/reference exists")
        _ref = _load_ref(p)
    return _ref


def host_has_avx512() -> bool:
    try:
        return "avx512f" in Path("/proc/cpuinfo").read_text()
    except OSError:
        return False


def REF_FAST():
    """Reference built with -O3 -march (paper flags) for CPU-baseline timing."""
    global _ref_fast
    if _ref_fast is None:
        name = "libevbref_v4.so" if host_has_avx512() else "libevbref_v3.so"
        p = REF_DIR / name
        if not p.exists():
            p = REF_DIR / "libevbref_exact.so"
        _ref_fast = _load_ref(p)
        _ref_fast._evb_name = p.name
    return _ref_fast


# ---- numpy helpers ------------------------------------------------------------------------------

def rng_words(seed: int, stream: int, n: int, skip: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    C().orc_rng_words(seed, stream, skip, n, ptr(out))
    return out


def philox_words(key: int, ctr_hi: int, start: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.uint64)
    C().orc_philox_words(key, ctr_hi, start, n, ptr(out))
    return out


def shift_rotation(seed: int, dim: int, stream: int = 1):
    o = np.empty(dim)
    m = np.empty(dim * dim)
    C().orc_make_shift_rotation(seed, stream, dim, ptr(o), ptr(m))
    return o, m.reshape(dim, dim)


def population(seed: int, pop: int, dim: int, stream: int = 2, lb: float = -100.0, ub: float = 100.0):
    x = np.empty((pop, dim))
    C().orc_init_population_seed(seed, stream, pop, dim, lb, ub, ptr(x))
    return x


def eval_batch(kind: int, shift, rot, bias: float, X) -> np.ndarray:
    """problems::evaluate_batch on a base instance, restated (fp64 or fp32 by X.dtype)."""
    X = np.ascontiguousarray(X)
    n, d = X.shape
    if X.dtype == np.float64:
        o = np.ascontiguousarray(shift, np.float64)
        m = np.ascontiguousarray(rot, np.float64)
        out = np.empty(n, np.float64)
        C().orc_eval_batch_f64(kind, d, ptr(o), ptr(m), bias, n, ptr(X), d, ptr(out))
    else:
        o = np.ascontiguousarray(shift, np.float32)
        m = np.ascontiguousarray(rot, np.float32)
        out = np.empty(n, np.float32)
        C().orc_eval_batch_f32(kind, d, ptr(o), ptr(m), np.float32(bias), n, ptr(X), d, ptr(out))
    return out


def eval_hybrid(shift, rot, bias, kinds, sizes, perm, X):
    X = np.ascontiguousarray(X)
    n, d = X.shape
    k = np.ascontiguousarray(kinds, np.int32)
    s = np.ascontiguousarray(sizes, np.int32)
    p = np.ascontiguousarray(perm, np.int32)
    if X.dtype == np.float64:
        o, m, out = np.ascontiguousarray(shift, np.float64), np.ascontiguousarray(rot, np.float64), np.empty(n)
        C().orc_eval_hybrid_f64(d, ptr(o), ptr(m), bias, len(k), ptr(k), ptr(s), ptr(p), n, ptr(X), d, ptr(out))
    else:
        o, m = np.ascontiguousarray(shift, np.float32), np.ascontiguousarray(rot, np.float32)
        out = np.empty(n, np.float32)
        C().orc_eval_hybrid_f32(d, ptr(o), ptr(m), np.float32(bias), len(k), ptr(k), ptr(s), ptr(p), n, ptr(X), d,
                                ptr(out))
    return out


def eval_composition(kinds, shifts, rots, sigma, lam, cbias, bias, X):
    X = np.ascontiguousarray(X)
    n, d = X.shape
    k = np.ascontiguousarray(kinds, np.int32)
    sg, la, cb = (np.ascontiguousarray(v, np.float64) for v in (sigma, lam, cbias))
    if X.dtype == np.float64:
        o, m, out = np.ascontiguousarray(shifts, np.float64), np.ascontiguousarray(rots, np.float64), np.empty(n)
        C().orc_eval_composition_f64(d, len(k), ptr(k), ptr(o), ptr(m), ptr(sg), ptr(la), ptr(cb), bias, n, ptr(X),
                                     d, ptr(out))
    else:
        o, m = np.ascontiguousarray(shifts, np.float32), np.ascontiguousarray(rots, np.float32)
        out = np.empty(n, np.float32)
        C().orc_eval_composition_f32(d, len(k), ptr(k), ptr(o), ptr(m), ptr(sg), ptr(la), ptr(cb), np.float32(bias),
                                     n, ptr(X), d, ptr(out))
    return out
