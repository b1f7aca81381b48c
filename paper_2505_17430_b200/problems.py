"""Host-side mirror of the reference problem interface over the C ABI.

Reference shapes kept:
  * ``ProblemInstance``   ~ ``problem_instance<T>``  (problems/instance.hpp:180-252), immutable,
                            device resident, shareable across tasks;
  * ``EvalScratch``       ~ ``eval_scratch<T>``      (problems/instance.hpp:45-56), per task;
  * ``evaluate_batch``    ~ ``problems::evaluate_batch(problem, xs, scratch, out)``
                            (problems/batch.hpp:243-278) on device tensors;
  * ``batched_evaluate``  ~ ``problems::batched_evaluate(problem, xs)`` (problems/batch.hpp:281-288)
                            on host arrays.
Errors map to the reference's: dimension mismatch -> ``InvalidArgument`` (std::invalid_argument),
configuration problems -> ``ConfigError`` (evobench::config_error).
"""
from __future__ import annotations

import ctypes
from enum import IntEnum
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import EVB_F32, EVB_F64, ConfigError, InvalidArgument, check


class BaseKind(IntEnum):
    """Same order as evobench::problems::base_kind (problems/functions.hpp:15-26)."""

    sphere = 0
    elliptic = 1
    bent_cigar = 2
    discus = 3
    rosenbrock = 4
    rastrigin = 5
    ackley = 6
    griewank = 7
    schwefel_12 = 8
    expanded_schaffer_f6 = 9


def _np_dtype(dtype: int):
    return np.float64 if dtype == EVB_F64 else np.float32


def dtype_of(x) -> int:
    name = str(getattr(x, "dtype", ""))
    if "float64" in name or name == "double":
        return EVB_F64
    if "float32" in name or name == "float":
        return EVB_F32
    raise ConfigError(f"unsupported dtype {name}")


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class ProblemInstance:
    """Immutable device-resident problem (problem_instance<T>)."""

    def __init__(self, handle: ctypes.c_void_p, dtype: int, dim: int, spec: str, kind: int | None, bias: float):
        self._h = handle
        self.dtype = dtype
        self.dim = dim
        self.spec = spec
        self.kind = kind
        self.bias = bias

    # --- constructors ---------------------------------------------------------------------
    @classmethod
    def base(cls, kind: int, shift, rotation, bias: float = 0.0, dtype: int = EVB_F64) -> "ProblemInstance":
        """Shifted-rotated base problem (problems/instance.hpp:185-196, 221-228)."""
        nd = _np_dtype(dtype)
        o = np.ascontiguousarray(shift, dtype=nd).reshape(-1)
        d = o.shape[0]
        m = np.ascontiguousarray(rotation, dtype=nd).reshape(-1)
        if m.shape[0] != d * d:
            raise ConfigError("problem: rotation must be dim x dim")
        h = ctypes.c_void_p()
        check(_lib.lib().evb_problem_create_base(dtype, d, int(kind), _ptr(o), _ptr(m), float(bias), ctypes.byref(h)),
              "evb_problem_create_base")
        return cls(h, dtype, d, "base", int(kind), float(bias))

    @classmethod
    def hybrid(cls, shift, rotation, sub_kinds: Sequence[int], chunk_sizes: Sequence[int], permutation: Sequence[int],
               bias: float = 0.0, dtype: int = EVB_F64) -> "ProblemInstance":
        """Hybrid problem (problems/instance.hpp:24-30, 97-112)."""
        nd = _np_dtype(dtype)
        o = np.ascontiguousarray(shift, dtype=nd).reshape(-1)
        d = o.shape[0]
        m = np.ascontiguousarray(rotation, dtype=nd).reshape(-1)
        k = np.ascontiguousarray(sub_kinds, dtype=np.int32)
        s = np.ascontiguousarray(chunk_sizes, dtype=np.int32)
        p = np.ascontiguousarray(permutation, dtype=np.int32)
        h = ctypes.c_void_p()
        check(_lib.lib().evb_problem_create_hybrid(dtype, d, _ptr(o), _ptr(m), float(bias), int(k.shape[0]), _ptr(k),
                                                   _ptr(s), _ptr(p), ctypes.byref(h)), "evb_problem_create_hybrid")
        return cls(h, dtype, d, "hybrid", None, float(bias))

    @classmethod
    def composition(cls, kinds: Sequence[int], shifts, rotations, sigma, lam, comp_bias, bias: float = 0.0,
                    dtype: int = EVB_F64) -> "ProblemInstance":
        """Composition problem (problems/instance.hpp:33-41, 116-174)."""
        nd = _np_dtype(dtype)
        k = np.ascontiguousarray(kinds, dtype=np.int32)
        n = k.shape[0]
        o = np.ascontiguousarray(shifts, dtype=nd).reshape(n, -1)
        d = o.shape[1]
        m = np.ascontiguousarray(rotations, dtype=nd).reshape(-1)
        if m.shape[0] != n * d * d:
            raise ConfigError("composition: rotations must be n_comp x dim x dim")
        sg = np.ascontiguousarray(sigma, dtype=np.float64)
        la = np.ascontiguousarray(lam, dtype=np.float64)
        cb = np.ascontiguousarray(comp_bias, dtype=np.float64)
        h = ctypes.c_void_p()
        check(_lib.lib().evb_problem_create_composition(dtype, d, n, _ptr(k), _ptr(o), _ptr(m), _ptr(sg), _ptr(la),
                                                        _ptr(cb), float(bias), ctypes.byref(h)),
              "evb_problem_create_composition")
        return cls(h, dtype, d, "composition", None, float(bias))

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise ConfigError("problem: already destroyed")
        return self._h

    def close(self) -> None:
        if self._h is not None:
            _lib.lib().evb_problem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class EvalScratch:
    """Per-task evaluation scratch (eval_scratch<T>); not shareable across concurrent streams."""

    def __init__(self):
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_scratch_create(ctypes.byref(self._h)), "evb_scratch_create")

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            _lib.lib().evb_scratch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev_ptr_and_ld(X, dim: int):
    """(pointer, n_rows, row stride) of a CUDA tensor holding points row-major."""
    if not getattr(X, "is_cuda", False):
        raise ConfigError("evaluate_batch: X must be a CUDA tensor (use batched_evaluate for host arrays)")
    if X.dim() != 2:
        raise InvalidArgument("evaluate_batch: X must be 2-D (points x dim)")
    if X.shape[0] > 0 and X.shape[1] != dim:
        raise InvalidArgument("evaluate_batch: point dimension mismatch")
    if X.stride(1) != 1:
        raise ConfigError("evaluate_batch: rows must be contiguous")
    ld = X.stride(0) if X.shape[0] > 1 else dim
    return ctypes.c_void_p(X.data_ptr()), int(X.shape[0]), int(max(ld, dim))


def _stream_ptr(stream):
    if stream is None:
        import torch

        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def evaluate_batch(problem: ProblemInstance, X, scratch: EvalScratch, out, stream=None) -> None:
    """out[b] = problem.evaluate(X[b]) on the device (problems/batch.hpp:243-278)."""
    if dtype_of(X) != problem.dtype or dtype_of(out) != problem.dtype:
        raise ConfigError("evaluate_batch: tensor dtype differs from the problem dtype")
    xp, n, ld = _dev_ptr_and_ld(X, problem.dim)
    if out.numel() < n:
        raise InvalidArgument("evaluate_batch: out is shorter than the batch")
    check(_lib.lib().evb_evaluate_batch(problem.handle, scratch.handle, xp, n, ld, ctypes.c_void_p(out.data_ptr()),
                                        _stream_ptr(stream)), "evaluate_batch")


def evaluate_batch_multi(problem: ProblemInstance, kinds: Sequence[int], biases: Sequence[float], X,
                         scratch: EvalScratch, out, stream=None) -> None:
    """Several base kinds on one z (BASELINE config 1); out is (len(kinds), n) row-major."""
    xp, n, ld = _dev_ptr_and_ld(X, problem.dim)
    k = (ctypes.c_int * len(kinds))(*[int(v) for v in kinds])
    b = (ctypes.c_double * len(biases))(*[float(v) for v in biases])
    ldo = out.stride(0) if out.dim() == 2 else n
    check(_lib.lib().evb_evaluate_batch_multi(problem.handle, scratch.handle, len(kinds), k, b, xp, n, ld,
                                              ctypes.c_void_p(out.data_ptr()), ldo, _stream_ptr(stream)),
          "evaluate_batch_multi")


def batched_evaluate(problem: ProblemInstance, xs, scratch: EvalScratch | None = None) -> np.ndarray:
    """Host-array convenience form (problems/batch.hpp:281-288): copies in, evaluates, copies out."""
    nd = _np_dtype(problem.dtype)
    x = np.ascontiguousarray(xs, dtype=nd)
    if x.size == 0:
        return np.zeros(0, dtype=nd)
    if x.ndim != 2 or x.shape[1] != problem.dim:
        raise InvalidArgument("evaluate_batch: point dimension mismatch")
    out = np.empty(x.shape[0], dtype=nd)
    sc = scratch or EvalScratch()
    check(_lib.lib().evb_evaluate_batch_host(problem.handle, sc.handle, _ptr(x), x.shape[0], x.shape[1], _ptr(out)),
          "batched_evaluate")
    return out


def batched_evaluate_many(problems: Sequence[ProblemInstance], xs, scratch: EvalScratch | None = None):
    """One host population on several problems (evb_evaluate_batch_host_many): X is copied to the
    device once; returns one fitness array per problem."""
    if not problems:
        return []
    nd = _np_dtype(problems[0].dtype)
    x = np.ascontiguousarray(xs, dtype=nd)
    if x.size == 0:
        return [np.zeros(0, dtype=nd) for _ in problems]
    if x.ndim != 2 or x.shape[1] != problems[0].dim:
        raise InvalidArgument("evaluate_batch: point dimension mismatch")
    outs = [np.empty(x.shape[0], dtype=nd) for _ in problems]
    handles = (ctypes.c_void_p * len(problems))(*[p.handle.value for p in problems])
    optrs = (ctypes.c_void_p * len(problems))(*[o.ctypes.data for o in outs])
    sc = scratch or EvalScratch()
    check(_lib.lib().evb_evaluate_batch_host_many(handles, len(problems), sc.handle, _ptr(x), x.shape[0], x.shape[1],
                                                  optrs), "batched_evaluate_many")
    return outs


def evaluate_batch_problems(problems: Sequence[ProblemInstance], X, scratch: EvalScratch, outs, stream=None) -> None:
    """One device population on several problems (evb_evaluate_batch_problems); outs[k] is a
    device vector for problem k.  Two or three fp64 base problems run as one launch."""
    xp, n, ld = _dev_ptr_and_ld(X, problems[0].dim)
    handles = (ctypes.c_void_p * len(problems))(*[p.handle.value for p in problems])
    optrs = (ctypes.c_void_p * len(problems))(*[o.data_ptr() for o in outs])
    check(_lib.lib().evb_evaluate_batch_problems(handles, len(problems), scratch.handle, xp, n, ld, optrs,
                                                 _stream_ptr(stream)), "evaluate_batch_problems")
