"""Host-side mirror of the reference PSO module (pso/engine.hpp, pso/topology.hpp, pso/update.hpp)
over the C ABI.  The GPU generation is SYNCHRONOUS (every particle reads the start-of-generation
personal bests); the stock reference engine is asynchronous (pso/engine.hpp:52-82) — see
DESIGN.md.  Positions, velocities and fitness are device tensors owned by the caller; personal
bests live in the engine, as in pso_engine<T>."""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import EVB_F32, EVB_F64, ConfigError, check
from .de import Rng, _sigs as _de_sigs
from .problems import EvalScratch, ProblemInstance, _stream_ptr, dtype_of

TOPOLOGIES = {"gbest": 0, "lbest_ring": 1}
UPDATES = {"standard": 0, "spherical": 1}


class _Cfg(ctypes.Structure):
    _fields_ = [("topology", ctypes.c_int), ("update", ctypes.c_int), ("inertia", ctypes.c_double),
                ("cognitive", ctypes.c_double), ("social", ctypes.c_double), ("vmax", ctypes.c_double),
                ("attraction", ctypes.c_double)]


@dataclass
class PSOConfig:
    """pso_builder slots + swarm_params (pso/update.hpp:16-22 defaults: SPSO2011 constants)."""

    topology: str = "gbest"
    update: str = "standard"
    inertia: float = 1.0 / (2.0 * math.log(2.0))
    cognitive: float = 0.5 + math.log(2.0)
    social: float = 0.5 + math.log(2.0)
    vmax: float = 0.0  # > 0: clamp |v| (BASELINE config 3: 0.2 * range = 40)
    attraction: float = 0.5 + math.log(2.0)  # spherical rule's c

    def to_c(self) -> _Cfg:
        if self.topology not in TOPOLOGIES:
            raise ConfigError(f"pso builder: unknown topology strategy '{self.topology}' (no GPU kernel)")
        if self.update not in UPDATES:
            raise ConfigError(f"pso builder: unknown update strategy '{self.update}' (no GPU kernel)")
        return _Cfg(TOPOLOGIES[self.topology], UPDATES[self.update], self.inertia, self.cognitive, self.social,
                    self.vmax, self.attraction)


def preset_spso2011() -> PSOConfig:
    """presets.hpp build_pso(spherical_ring = true): lbest ring + spherical update, SPSO2011 constants."""
    return PSOConfig("lbest_ring", "spherical")


def config3(topology: str) -> PSOConfig:
    """BASELINE config 3: w 0.7298, c1 = c2 = 1.49618, |v| <= 0.2 * (ub - lb) = 40."""
    return PSOConfig(topology, "standard", 0.7298, 1.49618, 1.49618, 40.0)


_REG = False


def _sigs():
    global _REG
    if _REG:
        return
    _de_sigs()
    P = ctypes.POINTER
    vp, i64, c_int, c_double, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint32
    _lib.register_signatures({
        "evb_pso_create": (c_int, [c_int, P(_Cfg), c_int, c_int, P(vp)]),
        "evb_pso_destroy": (c_int, [vp]),
        "evb_pso_prepare": (c_int, [vp, vp, i64, vp, vp]),
        "evb_pso_generation": (c_int, [vp, vp, vp, vp, i64, vp, i64, vp, c_double, c_double, vp, vp]),
        "evb_pso_init_uniform": (c_int, [vp, vp, i64, c_double, c_double, vp, vp]),
        "evb_pso_get": (c_int, [vp, vp, vp, vp, P(u32)]),
        "evb_pso_phase_timing": (c_int, [vp, c_int]),
        "evb_pso_phase_ms": (c_int, [vp, vp, c_int, P(c_int)]),
        "evb_pso_set_pbest": (c_int, [vp, vp, vp]),
        "evb_pso_optimize": (c_int, [vp, vp, vp, vp, i64, vp, i64, vp, c_double, c_double, i64, vp, P(c_int),
                                     P(c_double), P(c_int), vp]),
        "evb_pso_attach_recorder": (c_int, [vp, vp, c_int]),
    })
    _REG = True


class PSOEngine:
    def __init__(self, cfg: PSOConfig, pop_size: int, dim: int, dtype: int = EVB_F64):
        _sigs()
        self.cfg, self.pop_size, self.dim, self.dtype = cfg, pop_size, dim, dtype
        self._c = cfg.to_c()
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_pso_create(dtype, ctypes.byref(self._c), pop_size, dim, ctypes.byref(self._h)),
              "evb_pso_create")

    def _np(self):
        return np.float64 if self.dtype == EVB_F64 else np.float32

    def _chk(self, *ts):
        for t in ts:
            if dtype_of(t) != self.dtype:
                raise ConfigError("pso: tensor dtype differs from the engine dtype")

    def init_uniform(self, A, lo: float, hi: float, rng: Rng, stream=None) -> None:
        self._chk(A)
        check(_lib.lib().evb_pso_init_uniform(self._h, ctypes.c_void_p(A.data_ptr()), A.stride(0), lo, hi,
                                              rng.handle, _stream_ptr(stream)), "pso_init_uniform")

    def prepare(self, X, fitness, stream=None) -> None:
        self._chk(X, fitness)
        check(_lib.lib().evb_pso_prepare(self._h, ctypes.c_void_p(X.data_ptr()), X.stride(0),
                                         ctypes.c_void_p(fitness.data_ptr()), _stream_ptr(stream)), "pso_prepare")

    def generation(self, problem: ProblemInstance, X, V, fitness, lb: float, ub: float, rng: Rng,
                   scratch: EvalScratch | None = None, stream=None) -> None:
        self._chk(X, V, fitness)
        check(_lib.lib().evb_pso_generation(self._h, problem.handle, scratch.handle if scratch else None,
                                            ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(V.data_ptr()),
                                            V.stride(0), ctypes.c_void_p(fitness.data_ptr()), lb, ub, rng.handle,
                                            _stream_ptr(stream)), "pso_generation")

    def optimize(self, problem: ProblemInstance, X, V, fitness, lb: float, ub: float, max_fes: int, rng: Rng,
                 scratch: EvalScratch | None = None, stream=None):
        """pso_engine::optimize (pso/engine.hpp:84-105) with the synchronous generation."""
        self._chk(X, V, fitness)
        bi, bf, g = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        check(_lib.lib().evb_pso_optimize(self._h, problem.handle, scratch.handle if scratch else None,
                                          ctypes.c_void_p(X.data_ptr()), X.stride(0), ctypes.c_void_p(V.data_ptr()),
                                          V.stride(0), ctypes.c_void_p(fitness.data_ptr()), lb, ub, max_fes,
                                          rng.handle, ctypes.byref(bi), ctypes.byref(bf), ctypes.byref(g),
                                          _stream_ptr(stream)), "pso_optimize")
        return {"best_index": bi.value, "best_fitness": bf.value, "generations": g.value}

    def attach_recorder(self, recorder, run: int = 0) -> None:
        from .recorder import _sigs as _rec_sigs
        _rec_sigs()
        check(_lib.lib().evb_pso_attach_recorder(self._h, recorder.handle if recorder is not None else None, run),
              "pso_attach_recorder")
        self._recorder = recorder

    PHASES = ("neighbors", "update", "evaluate", "personal_best")

    def phase_timing(self, enable: bool = True) -> None:
        """Record CUDA events between the kernels of each later generation (bench accounting)."""
        check(_lib.lib().evb_pso_phase_timing(self._h, int(enable)), "pso_phase_timing")

    def phase_ms(self) -> dict:
        """Device time of each phase of the last generation (ms), synchronising on it."""
        ms = (ctypes.c_float * 8)()
        n = ctypes.c_int()
        check(_lib.lib().evb_pso_phase_ms(self._h, ms, 8, ctypes.byref(n)), "pso_phase_ms")
        return dict(zip(self.PHASES, [float(ms[k]) for k in range(n.value)]))

    def personal_bests(self):
        pb = np.zeros((self.pop_size, self.dim), self._np())
        pf = np.zeros(self.pop_size, self._np())
        nb = np.zeros(self.pop_size, np.int32)
        g = ctypes.c_uint32()
        check(_lib.lib().evb_pso_get(self._h, ctypes.c_void_p(pb.ctypes.data), ctypes.c_void_p(pf.ctypes.data),
                                     ctypes.c_void_p(nb.ctypes.data), ctypes.byref(g)), "pso_get")
        return {"pbest": pb, "pbest_fit": pf, "neighbors": nb, "generation": g.value}

    def set_personal_bests(self, pbest, pbest_fit) -> None:
        pb = np.ascontiguousarray(pbest, self._np())
        pf = np.ascontiguousarray(pbest_fit, self._np())
        check(_lib.lib().evb_pso_set_pbest(self._h, ctypes.c_void_p(pb.ctypes.data), ctypes.c_void_p(pf.ctypes.data)),
              "pso_set_pbest")

    def close(self):
        if self._h:
            _lib.lib().evb_pso_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scripted_words_for_generation(key: int, generation: int, pop_size: int, dim: int, philox=None,
                                  update: str = "standard"):
    """The sequential words the reference driver consumes for one Philox-mode PSO generation:
    particle i's sub-stream (g << 32) | i in particle order — 2*dim words (r1, r2 per gene) for the
    standard rule, 2*dim + 1 (dim normal pairs, then the radius uniform) for the spherical rule."""
    from .de import philox_words

    gen = philox or philox_words
    n = 2 * dim + (1 if update == "spherical" else 0)
    return np.concatenate([gen(key, (generation << 32) | i, 0, n) for i in range(pop_size)])
