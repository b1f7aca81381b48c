"""Competitive Swarm Optimizer (pso/cso.hpp:19-99, cso_optimizer<T>) over the C ABI.  A CSO
generation is data-parallel as the reference defines it (mean of the pre-update swarm, disjoint
random pairs, each loser reads only its winner), so the device generation IS the reference's
generation.  Positions, velocities and fitness are caller-owned device tensors."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import EVB_F64, ConfigError, check
from .de import Rng, _sigs as _de_sigs, philox_words
from .problems import EvalScratch, ProblemInstance, _stream_ptr, dtype_of

_REG = False


def _sigs():
    global _REG
    if _REG:
        return
    _de_sigs()
    from .recorder import _sigs as _rec_sigs
    _rec_sigs()
    P = ctypes.POINTER
    vp, i64, c_int, c_double = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double
    _lib.register_signatures({
        "evb_cso_create": (c_int, [c_int, c_double, c_int, c_int, P(vp)]),
        "evb_cso_destroy": (c_int, [vp]),
        "evb_cso_generation": (c_int, [vp, vp, vp, vp, i64, vp, i64, vp, c_double, c_double, vp, vp]),
        "evb_cso_optimize": (c_int, [vp, vp, vp, vp, i64, vp, i64, vp, c_double, c_double, i64, vp, P(c_int),
                                     P(c_double), P(c_int), vp]),
        "evb_cso_attach_recorder": (c_int, [vp, vp, c_int]),
    })
    _REG = True


class CSOEngine:
    """cso_optimizer<T>(phi) for pop_size particles of dimension dim."""

    def __init__(self, phi: float, pop_size: int, dim: int, dtype: int = EVB_F64):
        _sigs()
        self.phi, self.pop_size, self.dim, self.dtype = phi, pop_size, dim, dtype
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_cso_create(dtype, phi, pop_size, dim, ctypes.byref(self._h)), "cso_create")

    def _chk(self, X, V, fitness):
        for t in (X, V, fitness):
            if dtype_of(t) != self.dtype:
                raise ConfigError("cso: tensor dtype differs from the optimizer dtype")
        if tuple(X.shape) != (self.pop_size, self.dim) or tuple(V.shape) != (self.pop_size, self.dim):
            raise ConfigError("cso: X and V must be (pop_size, dim) CUDA tensors")
        return (ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(V.data_ptr()), V.stride(0),
                ctypes.c_void_p(fitness.data_ptr()))

    def generation(self, problem: ProblemInstance, X, V, fitness, lb: float, ub: float, rng: Rng,
                   scratch: EvalScratch | None = None, stream=None) -> None:
        x, ldx, v, ldv, f = self._chk(X, V, fitness)
        check(_lib.lib().evb_cso_generation(self._h, problem.handle, scratch.handle if scratch else None, x, ldx, v,
                                            ldv, f, lb, ub, rng.handle, _stream_ptr(stream)), "cso_generation")

    def optimize(self, problem: ProblemInstance, X, V, fitness, lb: float, ub: float, max_fes: int, rng: Rng,
                 scratch: EvalScratch | None = None, stream=None):
        x, ldx, v, ldv, f = self._chk(X, V, fitness)
        bi, bf, g = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        check(_lib.lib().evb_cso_optimize(self._h, problem.handle, scratch.handle if scratch else None, x, ldx, v,
                                          ldv, f, lb, ub, max_fes, rng.handle, ctypes.byref(bi), ctypes.byref(bf),
                                          ctypes.byref(g), _stream_ptr(stream)), "cso_optimize")
        return {"best_index": bi.value, "best_fitness": bf.value, "generations": g.value}

    def attach_recorder(self, recorder, run: int = 0) -> None:
        check(_lib.lib().evb_cso_attach_recorder(self._h, recorder.handle if recorder is not None else None, run),
              "cso_attach_recorder")
        self._recorder = recorder

    def close(self):
        if self._h:
            _lib.lib().evb_cso_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scripted_words_for_generation(key: int, generation: int, pop_size: int, dim: int, philox=None) -> np.ndarray:
    """The sequential words the reference's cso_optimizer::generation consumes for one Philox-mode
    device generation: the P-1 Fisher-Yates draws (sub-stream 0xFFFFFFFD), then pair t's 3*dim
    gene draws (sub-stream t) for t = 0 .. P/2-1."""
    gen_words = philox or philox_words
    parts = [gen_words(key, (generation << 32) | 0xFFFFFFFD, 0, pop_size - 1)]
    parts += [gen_words(key, (generation << 32) | t, 0, 3 * dim) for t in range(pop_size // 2)]
    return np.concatenate(parts)
