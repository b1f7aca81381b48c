"""Host-side mirror of the reference DE module (de/engine.hpp, de/builder.hpp, presets.hpp) over
the C ABI.  The engine owns per-run state (archive, adapter memories) exactly like
``de_engine<T>``; populations are device tensors ``(pop_size, dim)`` with a fitness vector.

Strategy slots are chosen by the reference's names; a slot without a GPU kernel raises
``ConfigError`` (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import EVB_F32, EVB_F64, ConfigError, check
from .problems import EvalScratch, ProblemInstance, _stream_ptr, dtype_of

MUTATIONS = {"rand_1": 0, "best_1": 1, "ttpb_1": 2}
CROSSOVERS = {"binomial": 0, "exponential": 1}
REPAIRS = {"clip": 0, "reflect": 1, "midpoint_target": 2, "reinitialize": 3}
POLICIES = {"fixed": 0, "linear_reduction": 1}
ADAPTERS = {"fixed": 0, "jade": 1, "shade": 2}


class _Cfg(ctypes.Structure):
    _fields_ = [("mutation", ctypes.c_int), ("crossover", ctypes.c_int), ("repair", ctypes.c_int),
                ("parameter", ctypes.c_int), ("f", ctypes.c_double), ("cr", ctypes.c_double),
                ("p_best", ctypes.c_double), ("use_archive", ctypes.c_int), ("memory_size", ctypes.c_int),
                ("jade_c", ctypes.c_double), ("archive_rate", ctypes.c_double), ("reduction", ctypes.c_int),
                ("n_min", ctypes.c_int)]


@dataclass
class DEConfig:
    """Slot choices of de_builder (de/builder.hpp:16-78)."""

    mutation: str = "rand_1"
    crossover: str = "binomial"
    repair: str = "clip"
    parameter: str = "fixed"
    f: float = 0.5
    cr: float = 0.9
    p_best: float = 0.11
    use_archive: bool = False
    memory_size: int = 1
    jade_c: float = 0.1
    archive_rate: float = 0.0
    reduction: str = "fixed"  # population_policy (de/policy.hpp): "fixed" | "linear_reduction"
    n_min: int = 4

    def to_c(self) -> _Cfg:
        for name, table, what in ((self.mutation, MUTATIONS, "mutation"), (self.crossover, CROSSOVERS, "crossover"),
                                  (self.repair, REPAIRS, "repair"), (self.parameter, ADAPTERS, "parameter adapter")):
            if name not in table:
                raise ConfigError(f"de builder: unknown {what} strategy '{name}' (no GPU kernel)")
        if self.reduction not in POLICIES:
            raise ConfigError(f"de builder: unknown population policy '{self.reduction}'")
        return _Cfg(MUTATIONS[self.mutation], CROSSOVERS[self.crossover], REPAIRS[self.repair],
                    ADAPTERS[self.parameter], self.f, self.cr, self.p_best, int(self.use_archive),
                    self.memory_size, self.jade_c, self.archive_rate, POLICIES[self.reduction], self.n_min)


def preset_de(f: float = 0.5, cr: float = 0.9) -> DEConfig:
    """presets.hpp:59-69 build_de_fixed: rand/1, binomial, clip, fixed(F, CR), archive 0."""
    return DEConfig("rand_1", "binomial", "clip", "fixed", f=f, cr=cr, archive_rate=0.0)


def preset_shade(p: float = 0.11, memory_size: int = 100, archive_rate: float = 1.0) -> DEConfig:
    """presets.hpp:83-94 build_shade: ttpb/1(p, archive), binomial, midpoint_target, shade(H)."""
    return DEConfig("ttpb_1", "binomial", "midpoint_target", "shade", p_best=p, use_archive=archive_rate > 0,
                    memory_size=memory_size, archive_rate=archive_rate)


def preset_lshade(p: float = 0.11, memory_size: int = 100, archive_rate: float = 1.0, n_min: int = 4) -> DEConfig:
    """presets.hpp:150-162 "lshade": build_shade with population_policy::linear_reduction(pop, n_min)."""
    return DEConfig("ttpb_1", "binomial", "midpoint_target", "shade", p_best=p, use_archive=archive_rate > 0,
                    memory_size=memory_size, archive_rate=archive_rate, reduction="linear_reduction", n_min=n_min)


def preset_jade(p: float = 0.05, c: float = 0.1, archive_rate: float = 0.0) -> DEConfig:
    """presets.hpp:71-81 build_jade: ttpb/1(p, archive), binomial, midpoint_target, jade(c)."""
    return DEConfig("ttpb_1", "binomial", "midpoint_target", "jade", p_best=p, use_archive=archive_rate > 0,
                    jade_c=c, archive_rate=archive_rate)


_SIGS = None


def _sigs():
    global _SIGS
    if _SIGS:
        return
    P = ctypes.POINTER
    vp, i64, c_int, c_double, u64, u32 = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_uint64, ctypes.c_uint32)
    _lib.register_signatures({
        "evb_rng_create_philox": (c_int, [u64, P(vp)]),
        "evb_rng_create_words": (c_int, [vp, i64, P(vp)]),
        "evb_rng_destroy": (c_int, [vp]),
        "evb_rng_state": (c_int, [vp, P(i64), P(u32), P(c_int)]),
        "evb_rng_set_generation": (c_int, [vp, u32]),
        "evb_philox_words": (c_int, [u64, u64, u64, i64, vp]),
        "evb_de_create": (c_int, [c_int, P(_Cfg), c_int, c_int, P(vp)]),
        "evb_de_destroy": (c_int, [vp]),
        "evb_de_reset": (c_int, [vp]),
        "evb_de_archive_capacity": (c_int, [vp]),
        "evb_de_p_count": (c_int, [vp]),
        "evb_de_pop_size": (c_int, [vp]),
        "evb_de_optimize_restart": (c_int, [vp, vp, vp, vp, i64, vp, c_double, c_double, i64, i64, c_double, vp,
                                            P(c_double), P(c_int), P(i64), vp]),
        "evb_de_set_budget": (c_int, [vp, i64, i64]),
        "evb_de_last_reduction": (c_int, [vp, P(c_int), P(c_int), P(i64)]),
        "evb_de_generation": (c_int, [vp, vp, vp, vp, i64, vp, c_double, c_double, vp, vp]),
        "evb_de_init_population": (c_int, [vp, vp, i64, c_double, c_double, vp, vp]),
        "evb_de_generations": (c_int, [vp, vp, vp, vp, i64, vp, c_double, c_double, vp, c_int, vp]),
        "evb_de_generations_host": (c_int, [vp, vp, vp, vp, i64, vp, c_double, c_double, vp, c_int]),
        "evb_de_optimize": (c_int, [vp, vp, vp, vp, i64, vp, c_double, c_double, i64, vp, P(c_int), P(c_double),
                                    P(c_int), vp]),
        "evb_de_get_state": (c_int, [vp, vp, P(c_int), vp, vp, P(c_int)]),
        "evb_de_set_state": (c_int, [vp, vp, c_int, vp, vp, c_int]),
        "evb_de_last_draws": (c_int, [vp, vp, P(i64), P(u32), vp, vp, vp, vp]),
        "evb_de_phase_timing": (c_int, [vp, c_int]),
        "evb_de_phase_ms": (c_int, [vp, vp, c_int, P(c_int)]),
    })
    _lib.lib()
    _SIGS = True


class Rng:
    """Device word source (core/rng.hpp semantics for every draw): Philox sub-streams or a
    caller-supplied word list consumed in the reference's sequential order (oracle mode)."""

    def __init__(self, handle, mode):
        self._h = handle
        self.mode = mode

    @classmethod
    def philox(cls, key: int) -> "Rng":
        _sigs()
        h = ctypes.c_void_p()
        check(_lib.lib().evb_rng_create_philox(ctypes.c_uint64(key), ctypes.byref(h)), "evb_rng_create_philox")
        return cls(h, "philox")

    @classmethod
    def words(cls, words) -> "Rng":
        _sigs()
        w = np.ascontiguousarray(words, dtype=np.uint64)
        h = ctypes.c_void_p()
        check(_lib.lib().evb_rng_create_words(ctypes.c_void_p(w.ctypes.data), w.shape[0], ctypes.byref(h)),
              "evb_rng_create_words")
        return cls(h, "words")

    @property
    def handle(self):
        return self._h

    def state(self):
        c, g, o = ctypes.c_int64(), ctypes.c_uint32(), ctypes.c_int()
        check(_lib.lib().evb_rng_state(self._h, ctypes.byref(c), ctypes.byref(g), ctypes.byref(o)), "rng_state")
        return {"cursor": c.value, "generation": g.value, "overflow": bool(o.value)}

    def set_generation(self, g: int) -> None:
        check(_lib.lib().evb_rng_set_generation(self._h, g), "rng_set_generation")

    def close(self):
        if self._h:
            _lib.lib().evb_rng_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def philox_words(key: int, ctr_hi: int, start: int, n: int) -> np.ndarray:
    """Device-generated Philox words (the exact stream the engines consume)."""
    _sigs()
    out = np.empty(n, dtype=np.uint64)
    check(_lib.lib().evb_philox_words(ctypes.c_uint64(key), ctypes.c_uint64(ctr_hi), ctypes.c_uint64(start), n,
                                      ctypes.c_void_p(out.ctypes.data)), "evb_philox_words")
    return out


class DEEngine:
    """de_engine<T> on the GPU (de/engine.hpp:71-173)."""

    def __init__(self, cfg: DEConfig, pop_size: int, dim: int, dtype: int = EVB_F64):
        _sigs()
        self.cfg = cfg
        self.pop_size = pop_size
        self.dim = dim
        self.dtype = dtype
        self._c = cfg.to_c()
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_de_create(dtype, ctypes.byref(self._c), pop_size, dim, ctypes.byref(self._h)),
              "evb_de_create")

    @property
    def archive_capacity(self) -> int:
        return int(_lib.lib().evb_de_archive_capacity(self._h))

    @property
    def p_count(self) -> int:
        return int(_lib.lib().evb_de_p_count(self._h))

    def reset(self) -> None:
        check(_lib.lib().evb_de_reset(self._h), "de_reset")

    def _pop(self, pop, fitness):
        if dtype_of(pop) != self.dtype or dtype_of(fitness) != self.dtype:
            raise ConfigError("de: tensor dtype differs from the engine dtype")
        if pop.dim() != 2 or pop.shape[0] < self.current_pop_size or pop.shape[1] != self.dim or pop.stride(1) != 1:
            raise ConfigError("de: population must be a (pop_size, dim) row-major CUDA tensor")
        return ctypes.c_void_p(pop.data_ptr()), pop.stride(0), ctypes.c_void_p(fitness.data_ptr())

    def generation(self, problem: ProblemInstance, pop, fitness, lb: float, ub: float, rng: Rng,
                   scratch: EvalScratch | None = None, stream=None) -> None:
        p, ld, f = self._pop(pop, fitness)
        check(_lib.lib().evb_de_generation(self._h, problem.handle, scratch.handle if scratch else None, p, ld, f,
                                           lb, ub, rng.handle, _stream_ptr(stream)), "de_generation")

    def generations(self, problem: ProblemInstance, pop, fitness, lb: float, ub: float, rng: Rng, n: int,
                    scratch: EvalScratch | None = None, stream=None) -> None:
        """n consecutive generations; after the first, a CUDA graph of one generation is replayed."""
        p, ld, f = self._pop(pop, fitness)
        check(_lib.lib().evb_de_generations(self._h, problem.handle, scratch.handle if scratch else None, p, ld, f,
                                            lb, ub, rng.handle, n, _stream_ptr(stream)), "de_generations")

    def generations_host(self, problem: ProblemInstance, pop: np.ndarray, fitness: np.ndarray, lb: float, ub: float,
                         rng: Rng, n: int, scratch: EvalScratch | None = None) -> None:
        """n generations on a host (numpy) population / fitness, updated in place: the reference's
        de_engine shape (one copy in, evb_de_generations, one copy out; synchronous)."""
        nd = self._np()
        if pop.dtype != nd or fitness.dtype != nd or pop.ndim != 2 or pop.shape[1] != self.dim \
                or pop.shape[0] != self.pop_size or pop.strides[1] != pop.itemsize \
                or pop.strides[0] % pop.itemsize or not fitness.flags["C_CONTIGUOUS"]:
            raise ConfigError("de: host population must be a row-major (pop_size, dim) array of the engine dtype")
        check(_lib.lib().evb_de_generations_host(self._h, problem.handle, scratch.handle if scratch else None,
                                                 ctypes.c_void_p(pop.ctypes.data), pop.strides[0] // pop.itemsize,
                                                 ctypes.c_void_p(fitness.ctypes.data), lb, ub, rng.handle, n),
              "de_generations_host")

    @property
    def current_pop_size(self) -> int:
        """Members after the last reduction (de/policy.hpp); rows [0, n) of the population."""
        return int(_lib.lib().evb_de_pop_size(self._h))

    def set_budget(self, max_fes: int, fes: int) -> None:
        """evolution_state(max_fes) with `fes` evaluations done (needed by linear_reduction)."""
        check(_lib.lib().evb_de_set_budget(self._h, max_fes, fes), "de_set_budget")

    def last_reduction(self):
        b, a, w = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        check(_lib.lib().evb_de_last_reduction(self._h, ctypes.byref(b), ctypes.byref(a), ctypes.byref(w)),
              "de_last_reduction")
        return {"pop_before": b.value, "pop_after": a.value, "shrink_words": w.value}

    def attach_param_trace(self, trace, run: int = 0) -> None:
        """Report (generation, mu_F, mu_CR) after every generation (parameter_record)."""
        from .recorder import _sigs as _rec_sigs
        _rec_sigs()
        check(_lib.lib().evb_de_attach_param_trace(self._h, trace.handle if trace is not None else None, run),
              "de_attach_param_trace")
        self._ptrace = trace

    def attach_recorder(self, recorder, run: int = 0) -> None:
        """Report every later evaluation (init inside optimize, each generation's trials, FE order)
        to `recorder` as run `run` (experiment/runner.hpp:38-52 run_handle). None detaches."""
        from .recorder import _sigs as _rec_sigs
        _rec_sigs()
        check(_lib.lib().evb_de_attach_recorder(self._h, recorder.handle if recorder is not None else None, run),
              "de_attach_recorder")
        self._recorder = recorder  # keep the device arrays alive while attached

    def init_population(self, pop, lb: float, ub: float, rng: Rng, stream=None) -> None:
        check(_lib.lib().evb_de_init_population(self._h, ctypes.c_void_p(pop.data_ptr()), pop.stride(0), lb, ub,
                                                rng.handle, _stream_ptr(stream)), "de_init_population")

    def optimize(self, problem: ProblemInstance, pop, fitness, lb: float, ub: float, max_fes: int, rng: Rng,
                 scratch: EvalScratch | None = None, stream=None):
        p, ld, f = self._pop(pop, fitness)
        bi, bf, g = ctypes.c_int(), ctypes.c_double(), ctypes.c_int()
        check(_lib.lib().evb_de_optimize(self._h, problem.handle, scratch.handle if scratch else None, p, ld, f, lb,
                                         ub, max_fes, rng.handle, ctypes.byref(bi), ctypes.byref(bf),
                                         ctypes.byref(g), _stream_ptr(stream)), "de_optimize")
        return {"best_index": bi.value, "best_fitness": bf.value, "generations": g.value}

    def optimize_restart(self, problem: ProblemInstance, pop, fitness, lb: float, ub: float, total_budget: int,
                         stagnation_evals: int, epsilon: float, rng: Rng, scratch: EvalScratch | None = None,
                         stream=None):
        """hybrid::restart_run around this engine (the "restart-lshade" preset with an L-SHADE
        configuration): fresh engine states until the budget is spent."""
        p, ld, f = self._pop(pop, fitness)
        bf, runs, ev = ctypes.c_double(), ctypes.c_int(), ctypes.c_int64()
        check(_lib.lib().evb_de_optimize_restart(self._h, problem.handle, scratch.handle if scratch else None, p, ld, f,
                                                 lb, ub, total_budget, stagnation_evals, epsilon, rng.handle,
                                                 ctypes.byref(bf), ctypes.byref(runs), ctypes.byref(ev),
                                                 _stream_ptr(stream)), "de_optimize_restart")
        return {"best_fitness": bf.value, "engine_runs": runs.value, "evaluations": ev.value}

    def _np(self):
        return np.float64 if self.dtype == EVB_F64 else np.float32

    def get_state(self):
        cap = max(1, self.archive_capacity)
        H = max(1, self.cfg.memory_size if self.cfg.parameter == "shade" else 1)
        arch = np.zeros((cap, self.dim), self._np())
        mf = np.zeros(H, self._np())
        mc = np.zeros(H, self._np())
        sz, wi = ctypes.c_int(), ctypes.c_int()
        check(_lib.lib().evb_de_get_state(self._h, ctypes.c_void_p(arch.ctypes.data), ctypes.byref(sz),
                                          ctypes.c_void_p(mf.ctypes.data), ctypes.c_void_p(mc.ctypes.data),
                                          ctypes.byref(wi)), "de_get_state")
        return {"archive": arch[:sz.value], "archive_size": sz.value, "memory_f": mf, "memory_cr": mc,
                "write_index": wi.value}

    def set_state(self, archive, memory_f, memory_cr, write_index: int) -> None:
        a = np.ascontiguousarray(archive, self._np()).reshape(-1, self.dim)
        mf = np.ascontiguousarray(memory_f, self._np())
        mc = np.ascontiguousarray(memory_cr, self._np())
        check(_lib.lib().evb_de_set_state(self._h, ctypes.c_void_p(a.ctypes.data), a.shape[0],
                                          ctypes.c_void_p(mf.ctypes.data), ctypes.c_void_p(mc.ctypes.data),
                                          write_index), "de_set_state")

    PHASES = ("order", "draws", "trial", "evaluate", "select_scan", "select_apply")

    def phase_timing(self, enable: bool = True) -> None:
        """Record CUDA events between the kernels of each later generation (bench accounting)."""
        check(_lib.lib().evb_de_phase_timing(self._h, int(enable)), "de_phase_timing")

    def phase_ms(self) -> dict:
        """Device time of each phase of the last generation (ms), synchronising on it."""
        ms = (ctypes.c_float * 8)()
        n = ctypes.c_int()
        check(_lib.lib().evb_de_phase_ms(self._h, ms, 8, ctypes.byref(n)), "de_phase_ms")
        return dict(zip(self.PHASES, [float(ms[k]) for k in range(n.value)]))

    def last_draws(self):
        P = self.pop_size
        wc = np.zeros(P, np.int64)
        aw = ctypes.c_int64()
        gen = ctypes.c_uint32()
        F = np.zeros(P, self._np())
        CR = np.zeros(P, self._np())
        idx = np.zeros((P, 4), np.int32)
        jr = np.zeros(P, np.int32)
        check(_lib.lib().evb_de_last_draws(self._h, ctypes.c_void_p(wc.ctypes.data), ctypes.byref(aw),
                                           ctypes.byref(gen), ctypes.c_void_p(F.ctypes.data),
                                           ctypes.c_void_p(CR.ctypes.data), ctypes.c_void_p(idx.ctypes.data),
                                           ctypes.c_void_p(jr.ctypes.data)), "de_last_draws")
        n = self.last_reduction()["pop_before"] or P
        return {"word_counts": wc[:n], "archive_words": aw.value, "generation": gen.value, "F": F[:n], "CR": CR[:n],
                "idx": idx[:n], "jrand": jr[:n]}

    def close(self):
        if self._h:
            _lib.lib().evb_de_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def scripted_words_for_generation(key: int, generation: int, word_counts, archive_words: int, philox=None,
                                  shrink_words: int = 0):
    """The sequential word list the reference engine consumes for one Philox-mode generation:
    individual i's sub-stream prefix (word_counts[i] words) in i order, then the archive-victim
    words, then (population reduction) the archive-shrink words.  ``philox(key, ctr_hi, start,
    n)`` generates words (default: the device generator)."""
    gen_words = philox or philox_words
    parts = [gen_words(key, (generation << 32) | i, 0, int(c)) for i, c in enumerate(word_counts)]
    if archive_words:
        parts.append(gen_words(key, (generation << 32) | 0xFFFFFFFF, 0, int(archive_words)))
    if shrink_words:
        parts.append(gen_words(key, (generation << 32) | 0xFFFFFFFE, 0, int(shrink_words)))
    return np.concatenate(parts) if parts else np.zeros(0, np.uint64)
