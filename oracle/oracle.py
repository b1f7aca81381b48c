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


# ---- DE: the reference engine (REF) and the C restatement (C) -------------------------------------
REF_DE_SIG = {
    "ref_de_create": (vp, [c_int, c_int, c_int, c_double, c_double, c_double, c_int, c_int, c_double, c_double,
                           c_int, c_int, c_int, c_int, c_int]),
    "ref_de_set_budget": (None, [vp, ctypes.c_longlong, ctypes.c_longlong]),
    "ref_de_pop_size": (c_int, [vp]),
    "ref_de_destroy": (None, [vp]),
    "ref_de_set_problem_base": (None, [vp, c_int, vp, vp, c_double]),
    "ref_de_set_problem_composition": (None, [vp, c_int, vp, vp, vp, vp, vp, vp, c_double]),
    "ref_de_set_pop": (None, [vp, vp, vp]),
    "ref_de_init": (i64, [vp, vp, i64, c_double, c_double]),
    "ref_de_generation": (c_int, [vp, vp, i64, c_double, c_double]),
    "ref_de_get": (None, [vp, vp, vp, vp, vp, vp, vp, vp]),
    "ref_de_native_run": (None, [vp, u64, u64, c_int, c_double, c_double]),
}
register_ref(REF_DE_SIG)

MUT = {"rand_1": 0, "best_1": 1, "ttpb_1": 2}
REP = {"clip": 0, "reflect": 1, "midpoint_target": 2, "reinitialize": 3}
CX = {"binomial": 0, "exponential": 1}
ADA = {"fixed": 0, "jade": 1, "shade": 2}


class RefDE:
    """The reference de_engine<double> (built through de_builder) stepped one generation at a
    time with rng_stream::scripted word lists (or run natively)."""

    def __init__(self, cfg, P, D):
        self.P, self.D, self.cfg = P, D, cfg
        self.H = max(1, cfg.memory_size if cfg.parameter == "shade" else 1)
        self.h = REF().ref_de_create(MUT[cfg.mutation], REP[cfg.repair], ADA[cfg.parameter], cfg.f, cfg.cr,
                                     cfg.p_best, int(cfg.use_archive), self.H, cfg.jade_c, cfg.archive_rate, P, D,
                                     CX[cfg.crossover], int(cfg.reduction == "linear_reduction"), cfg.n_min)
        self._keep = []

    def set_problem_base(self, kind, shift, rot, bias):
        o = np.ascontiguousarray(shift, np.float64)
        m = np.ascontiguousarray(rot, np.float64).ravel()
        self._keep += [o, m]
        REF().ref_de_set_problem_base(self.h, int(kind), ptr(o), ptr(m), bias)

    def set_problem_composition(self, kinds, shifts, rots, sigma, lam, cbias, bias=0.0):
        arrs = [np.ascontiguousarray(kinds, np.int32), np.ascontiguousarray(shifts, np.float64),
                np.ascontiguousarray(rots, np.float64), np.ascontiguousarray(sigma, np.float64),
                np.ascontiguousarray(lam, np.float64), np.ascontiguousarray(cbias, np.float64)]
        self._keep += arrs
        REF().ref_de_set_problem_composition(self.h, len(arrs[0]), *[ptr(a) for a in arrs], bias)

    def set_pop(self, x, fit):
        x = np.ascontiguousarray(x, np.float64)
        f = np.ascontiguousarray(fit, np.float64)
        REF().ref_de_set_pop(self.h, ptr(x), ptr(f))

    def init(self, words, lb, ub):
        w = np.ascontiguousarray(words, np.uint64)
        return int(REF().ref_de_init(self.h, ptr(w), len(w), lb, ub))

    def generation(self, words, lb, ub) -> bool:
        w = np.ascontiguousarray(words, np.uint64)
        return bool(REF().ref_de_generation(self.h, ptr(w), len(w), lb, ub))

    def native_run(self, seed, stream, generations, lb, ub):
        REF().ref_de_native_run(self.h, seed, stream, generations, lb, ub)

    def set_budget(self, max_fes, fes):
        REF().ref_de_set_budget(self.h, max_fes, fes)

    def pop_size(self):
        return int(REF().ref_de_pop_size(self.h))

    def get(self):
        n = self.pop_size()
        x = np.empty((n, self.D))
        f = np.empty(n)
        cap = max(1, int(np.ceil(self.cfg.archive_rate * self.P)))
        a = np.zeros((cap, self.D))
        sz, wi = ctypes.c_int(), ctypes.c_int()
        mf = np.zeros(self.H)
        mc = np.zeros(self.H)
        REF().ref_de_get(self.h, ptr(x), ptr(f), ptr(a), ctypes.byref(sz), ptr(mf), ptr(mc), ctypes.byref(wi))
        return {"pop": x, "fit": f, "archive": a[:sz.value], "archive_size": sz.value, "memory_f": mf,
                "memory_cr": mc, "write_index": wi.value}

    def __del__(self):
        try:
            REF().ref_de_destroy(self.h)
        except Exception:
            pass


class _OrcDeCfg(ctypes.Structure):
    _fields_ = [("mutation", c_int), ("repair", c_int), ("parameter", c_int), ("f", c_double), ("cr", c_double),
                ("p", c_double), ("use_archive", c_int), ("H", c_int), ("jade_c", c_double), ("P", c_int),
                ("D", c_int), ("archive_cap", c_int), ("kind", c_int), ("shift", vp), ("rot", vp),
                ("bias", c_double), ("n_comp", c_int), ("comp_kinds", vp), ("comp_shifts", vp), ("comp_rots", vp),
                ("sigma", vp), ("lambda_", vp), ("cbias", vp), ("crossover", c_int)]


class _OrcDeState(ctypes.Structure):
    _fields_ = [("pop", vp), ("fit", vp), ("archive", vp), ("arch_size", c_int), ("mem_f", vp), ("mem_cr", vp),
                ("write_index", c_int)]


register_c({
    "orc_de_generation": (i64, [ctypes.POINTER(_OrcDeCfg), ctypes.POINTER(_OrcDeState), vp, c_double, c_double, vp,
                                vp, vp, vp, vp, vp]),
    "orc_de_cfg_size": (c_int, []),
    "orc_de_state_size": (c_int, []),
})


class OracleDE:
    """The C restatement of de_engine::generation (oracle/evb_oracle.c), exporting the integer
    outputs (donor indices, jrand, selection mask, words per individual)."""

    def __init__(self, cfg, P, D):
        assert C().orc_de_cfg_size() == ctypes.sizeof(_OrcDeCfg)
        self.cfg, self.P, self.D = cfg, P, D
        self.H = max(1, cfg.memory_size if cfg.parameter == "shade" else 1)
        self.cap = int(np.ceil(cfg.archive_rate * P))
        self.c = _OrcDeCfg(MUT[cfg.mutation], REP[cfg.repair], ADA[cfg.parameter], cfg.f, cfg.cr, cfg.p_best,
                           int(cfg.use_archive), self.H, cfg.jade_c, P, D, self.cap)
        self.c.kind = -1
        self.c.crossover = CX[cfg.crossover]
        self.pop = np.zeros((P, D))
        self.fit = np.zeros(P)
        self.archive = np.zeros((max(1, self.cap), D))
        self.mem_f = np.full(self.H, 0.5)
        self.mem_cr = np.full(self.H, 0.5)
        self.s = _OrcDeState(ptr(self.pop), ptr(self.fit), ptr(self.archive), 0, ptr(self.mem_f), ptr(self.mem_cr), 0)
        self._keep = []

    def set_problem_base(self, kind, shift, rot, bias):
        o = np.ascontiguousarray(shift, np.float64)
        m = np.ascontiguousarray(rot, np.float64).ravel()
        self._keep += [o, m]
        self.c.kind, self.c.shift, self.c.rot, self.c.bias = int(kind), o.ctypes.data, m.ctypes.data, bias

    def set_problem_composition(self, kinds, shifts, rots, sigma, lam, cbias, bias=0.0):
        arrs = [np.ascontiguousarray(kinds, np.int32), np.ascontiguousarray(shifts, np.float64),
                np.ascontiguousarray(rots, np.float64), np.ascontiguousarray(sigma, np.float64),
                np.ascontiguousarray(lam, np.float64), np.ascontiguousarray(cbias, np.float64)]
        self._keep += arrs
        self.c.n_comp = len(arrs[0])
        (self.c.comp_kinds, self.c.comp_shifts, self.c.comp_rots, self.c.sigma, self.c.lambda_,
         self.c.cbias) = [a.ctypes.data for a in arrs]
        self.c.bias = bias

    def set_state(self, pop, fit, archive=None, arch_size=0, mem_f=None, mem_cr=None, write_index=0):
        self.pop[:] = pop
        self.fit[:] = fit
        if archive is not None and arch_size:
            self.archive[:arch_size] = archive[:arch_size]
        self.s.arch_size = arch_size
        if mem_f is not None:
            self.mem_f[:] = mem_f
            self.mem_cr[:] = mem_cr
        self.s.write_index = write_index

    def generation(self, words, lb, ub):
        w = np.ascontiguousarray(words, np.uint64)
        rng = ctypes.create_string_buffer(C().orc_rng_size())
        C().orc_rng_scripted(rng, ptr(w), len(w))
        P = self.P
        out = {"F": np.zeros(P), "CR": np.zeros(P), "idx": np.zeros((P, 4), np.int32), "jrand": np.zeros(P, np.int32),
               "words": np.zeros(P, np.int64), "win": np.zeros(P, np.int32)}
        aw = C().orc_de_generation(ctypes.byref(self.c), ctypes.byref(self.s), rng, lb, ub, ptr(out["F"]),
                                   ptr(out["CR"]), ptr(out["idx"]), ptr(out["jrand"]), ptr(out["words"]),
                                   ptr(out["win"]))
        out["archive_words"] = int(aw)
        return out


# ---- PSO: synchronous driver over the reference pieces (REF) and the C restatement (C) ------------
register_ref({
    "ref_pso_create": (vp, [c_int, c_int, c_double, c_double, c_double, c_double, c_int, c_int, c_int, vp, vp,
                            c_double, c_int, c_double]),
    "ref_pso_set": (None, [c_int, vp, vp, vp, vp]),
    "ref_pso_step": (c_int, [c_int, vp, vp, i64, c_double, c_double]),
    "ref_pso_get": (None, [c_int, vp, vp, vp, vp, vp, vp]),
    "ref_pso_destroy": (None, [c_int, vp]),
})
_PSO_C = {"orc_pso_step_f64": (None, [c_int, c_double, c_double, c_double, c_double, c_int, c_int, c_int, vp, vp,
                                      c_double, vp, vp, vp, vp, vp, vp, i64, c_double, c_double, vp]),
          "orc_pso_step_f32": (None, [c_int, c_double, c_double, c_double, c_double, c_int, c_int, c_int, vp, vp,
                                      c_float, vp, vp, vp, vp, vp, vp, i64, c_float, c_float, vp])}
register_c(_PSO_C)


class RefPSO:
    def __init__(self, dtype_np, topology, w, c1, c2, vmax, P, D, kind, shift, rot, bias=0.0, update=0,
                 attraction=0.0):
        self.nd = dtype_np
        self.dt = 1 if dtype_np == np.float64 else 0
        self.P, self.D = P, D
        self._o = np.ascontiguousarray(shift, dtype_np)
        self._m = np.ascontiguousarray(rot, dtype_np).ravel()
        self.h = REF().ref_pso_create(self.dt, topology, w, c1, c2, vmax, P, D, kind, ptr(self._o), ptr(self._m), bias,
                                      update, attraction)

    def set(self, x, v, fit):
        x, v, f = (np.ascontiguousarray(a, self.nd) for a in (x, v, fit))
        REF().ref_pso_set(self.dt, self.h, ptr(x), ptr(v), ptr(f))

    def step(self, words, lb, ub) -> bool:
        w = np.ascontiguousarray(words, np.uint64)
        return bool(REF().ref_pso_step(self.dt, self.h, ptr(w), len(w), lb, ub))

    def set_threads(self, n: int) -> None:
        """Evaluate the swarm on n host threads (contiguous slices, one eval_scratch each)."""
        REF().ref_pso_set_threads(self.dt, self.h, int(n))

    def get(self):
        P, D = self.P, self.D
        out = {k: np.zeros((P, D), self.nd) for k in ("x", "v", "pbest")}
        out["fit"] = np.zeros(P, self.nd)
        out["pbest_fit"] = np.zeros(P, self.nd)
        REF().ref_pso_get(self.dt, self.h, ptr(out["x"]), ptr(out["v"]), ptr(out["fit"]), ptr(out["pbest"]),
                          ptr(out["pbest_fit"]))
        return out

    def __del__(self):
        try:
            REF().ref_pso_destroy(self.dt, self.h)
        except Exception:
            pass


def pso_step_c(topology, w, c1, c2, vmax, kind, shift, rot, bias, x, v, fit, pb, pbf, words, lb, ub):
    """C restatement, in place on numpy arrays; returns the neighbour index of every particle."""
    nd = x.dtype
    P, D = x.shape
    o = np.ascontiguousarray(shift, nd)
    m = np.ascontiguousarray(rot, nd).ravel()
    w_ = np.ascontiguousarray(words, np.uint64)
    nb = np.zeros(P, np.int32)
    fn = C().orc_pso_step_f64 if nd == np.float64 else C().orc_pso_step_f32
    fn(topology, w, c1, c2, vmax, P, D, kind, ptr(o), ptr(m), bias, ptr(x), ptr(v), ptr(fit), ptr(pb), ptr(pbf),
       ptr(w_), len(w_), lb, ub, ptr(nb))
    return nb


register_c({"orc_de_fixed_generation_words": (i64, [c_int, u64, ctypes.c_uint32, c_int, c_int, vp, i64])})


def de_fixed_generation_words(mutation: int, key: int, gen: int, P: int, D: int) -> np.ndarray:
    cap = P * (D + 64)
    out = np.empty(cap, np.uint64)
    n = C().orc_de_fixed_generation_words(mutation, key, gen, P, D, ptr(out), cap)
    assert n <= cap
    return out[:n].copy()


register_c({"orc_make_composition": (None, [u64, u64, c_int, c_int, vp, vp])})
register_ref({"ref_make_composition": (None, [u64, u64, c_int, c_int, vp, vp])})

# BASELINE config 4 composition recipe (component order: Rastrigin, elliptic, Ackley)
CONFIG4_KINDS = [5, 1, 6]
CONFIG4_SIGMA = [10.0, 20.0, 30.0]
CONFIG4_LAMBDA = [1.0, 1e-6, 1.0]
CONFIG4_BIAS = [0.0, 100.0, 200.0]


def composition_components(seed: int, dim: int, n_comp: int = 3, stream: int = 1):
    s = np.empty((n_comp, dim))
    m = np.empty((n_comp, dim, dim))
    C().orc_make_composition(seed, stream, dim, n_comp, ptr(s), ptr(m))
    return s, m


register_ref({
    "ref_pso_set_threads": (None, [c_int, vp, c_int]),
    "ref_bench_config4": (c_double, [c_int, c_int, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp]),
    "ref_bench_de": (c_double, [c_int, c_int, c_int, c_int, c_int, vp, vp, u64]),
})


register_ref({
    "ref_record": (i64, [vp, c_int, vp, c_int, c_int, ctypes.c_longlong, ctypes.c_longlong, vp, vp, i64]),
    "ref_de_generation_trace": (c_int, [vp, vp, i64, c_double, c_double, vp]),
})


def ref_record(values_per_run, dim: int, max_fes: int, interval: int):
    """The reference best_so_far_record fed with each run's values in FE order (+ on_run_end);
    returns (grid, csv)."""
    runs = len(values_per_run)
    n = max(1, max(len(v) for v in values_per_run))
    vals = np.full((runs, n), np.nan)
    for r, v in enumerate(values_per_run):
        vals[r, :len(v)] = v
    counts = np.array([len(v) for v in values_per_run], np.int32)
    ck = max_fes // interval
    grid = np.zeros((runs, ck))
    ln = REF().ref_record(ptr(vals), n, ptr(counts), runs, dim, max_fes, interval, ptr(grid), None, 0)
    buf = ctypes.create_string_buffer(int(ln) + 1)
    REF().ref_record(ptr(vals), n, ptr(counts), runs, dim, max_fes, interval, ptr(grid), buf, int(ln))
    return grid, buf.raw[:ln].decode()


def _refde_generation_trace(self, words, lb, ub):
    w = np.ascontiguousarray(words, np.uint64)
    vals = np.empty(self.P)
    ok = bool(REF().ref_de_generation_trace(self.h, ptr(w), len(w), lb, ub, ptr(vals)))
    return ok, vals


RefDE.generation_trace = _refde_generation_trace


register_ref({"ref_de_native_trace": (None, [vp, ctypes.c_uint64, ctypes.c_uint64, c_int, c_double, c_double, vp])})


def _refde_native_trace(self, seed, stream, generations, lb, ub):
    vals = np.empty(self.P * (generations + 1))
    REF().ref_de_native_trace(self.h, seed, stream, generations, lb, ub, ptr(vals))
    return vals


RefDE.native_trace = _refde_native_trace


register_ref({"ref_evo_bench_de": (i64, [c_double, c_double, c_int, c_int, c_int, vp, c_int, c_int, ctypes.c_longlong,
                                         ctypes.c_longlong, vp, vp, vp, c_double, vp, vp, c_double, c_double, c_int,
                                         vp, i64, vp])})


def de_task_words(key: int, P: int, D: int, generations: int, mutation: int = 0) -> np.ndarray:
    """The words a task's positional Philox stream yields in the reference's consumption order:
    init_population (sub-stream 0xFFFFFFF0 of generation 0), then generations 1..G."""
    parts = [philox_words(key, 0xFFFFFFF0, 0, P * D)]
    for g in range(1, generations + 1):
        parts.append(de_fixed_generation_words(mutation, key, g, P, D))
    return np.concatenate(parts)


def ref_evo_bench_de(f, cr, P, D, problem_ids, instances, runs, max_fes, interval, kinds, shifts, rots, bias,
                     task_words, lb=-100.0, ub=100.0, threads=0):
    """experiment::evo_bench with the `de` preset over a suite of base problems, the reference's
    recorder attached; task t replays task_words[t].  Returns (csv, best per task)."""
    n_problems = len(problem_ids)
    ids = np.ascontiguousarray(problem_ids, np.int32)
    k = np.ascontiguousarray(kinds, np.int32)
    sh = np.ascontiguousarray(shifts, np.float64)
    ro = np.ascontiguousarray(rots, np.float64)
    words = np.ascontiguousarray(np.concatenate(task_words), np.uint64)
    off = np.zeros(len(task_words) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in task_words])
    best = np.zeros(len(task_words))
    args = (f, cr, P, D, n_problems, ptr(ids), instances, runs, max_fes, interval, ptr(k), ptr(sh), ptr(ro), bias,
            ptr(words), ptr(off), lb, ub, threads)
    n = REF().ref_evo_bench_de(*args, None, 0, ptr(best))
    buf = ctypes.create_string_buffer(int(n) + 1)
    REF().ref_evo_bench_de(*args, buf, int(n), ptr(best))
    return buf.raw[:n].decode(), best


register_ref({
    "ref_cso_create": (vp, [c_int, c_double, c_int, c_int, c_int, vp, vp, c_double]),
    "ref_cso_set": (None, [c_int, vp, vp, vp, vp]),
    "ref_cso_step": (c_int, [c_int, vp, vp, i64, c_double, c_double]),
    "ref_cso_get": (None, [c_int, vp, vp, vp, vp]),
    "ref_cso_native_optimize": (c_double, [c_int, vp, ctypes.c_uint64, ctypes.c_uint64, c_double, c_double,
                                           ctypes.c_longlong]),
    "ref_cso_destroy": (None, [c_int, vp]),
})


class RefCSO:
    """The reference's cso_optimizer<T> (pso/cso.hpp) stepped with scripted words."""

    def __init__(self, phi, P, D, kind, shift, rot, bias=0.0, dtype=np.float64):
        self.nd = np.dtype(dtype)
        self.dt = 1 if self.nd == np.float64 else 0
        self.P, self.D = P, D
        self._o = np.ascontiguousarray(shift, self.nd)
        self._m = np.ascontiguousarray(rot, self.nd).ravel()
        self.h = REF().ref_cso_create(self.dt, phi, P, D, kind, ptr(self._o), ptr(self._m), bias)

    def set(self, x, v, fit):
        x = np.ascontiguousarray(x, self.nd)
        v = np.ascontiguousarray(v, self.nd)
        f = np.ascontiguousarray(fit, self.nd)
        REF().ref_cso_set(self.dt, self.h, ptr(x), ptr(v), ptr(f))

    def step(self, words, lb, ub) -> bool:
        w = np.ascontiguousarray(words, np.uint64)
        return bool(REF().ref_cso_step(self.dt, self.h, ptr(w), len(w), lb, ub))

    def get(self):
        x = np.zeros((self.P, self.D), self.nd)
        v = np.zeros((self.P, self.D), self.nd)
        f = np.zeros(self.P, self.nd)
        REF().ref_cso_get(self.dt, self.h, ptr(x), ptr(v), ptr(f))
        return {"x": x, "v": v, "fit": f}

    def native_optimize(self, seed, stream, lb, ub, max_fes):
        return float(REF().ref_cso_native_optimize(self.dt, self.h, seed, stream, lb, ub, max_fes))

    def __del__(self):
        try:
            REF().ref_cso_destroy(self.dt, self.h)
        except Exception:
            pass


register_ref({"ref_evo_bench_cso": (i64, [c_double, c_int, c_int, c_int, vp, c_int, c_int, ctypes.c_longlong,
                                          ctypes.c_longlong, vp, vp, vp, c_double, vp, vp, c_double, c_double, c_int,
                                          vp, i64, vp])})


def ref_evo_bench_cso(phi, P, D, problem_ids, instances, runs, max_fes, interval, kinds, shifts, rots, bias,
                      task_words, lb=-100.0, ub=100.0, threads=0):
    """experiment::evo_bench with the `cso` preset, the reference recorder attached; task t replays
    task_words[t].  Returns (csv, best per task)."""
    ids = np.ascontiguousarray(problem_ids, np.int32)
    k = np.ascontiguousarray(kinds, np.int32)
    sh = np.ascontiguousarray(shifts, np.float64)
    ro = np.ascontiguousarray(rots, np.float64)
    words = np.ascontiguousarray(np.concatenate(task_words), np.uint64)
    off = np.zeros(len(task_words) + 1, np.int64)
    off[1:] = np.cumsum([len(w) for w in task_words])
    best = np.zeros(len(task_words))
    args = (phi, P, D, len(ids), ptr(ids), instances, runs, max_fes, interval, ptr(k), ptr(sh), ptr(ro), bias,
            ptr(words), ptr(off), lb, ub, threads)
    n = REF().ref_evo_bench_cso(*args, None, 0, ptr(best))
    buf = ctypes.create_string_buffer(int(n) + 1)
    REF().ref_evo_bench_cso(*args, buf, int(n), ptr(best))
    return buf.raw[:n].decode(), best


register_ref({
    "ref_de_params": (c_int, [vp, vp, vp]),
    "ref_param_record": (i64, [vp, vp, vp, c_int, vp, c_int, vp, c_int, c_int, c_int, vp, i64]),
})


def _refde_params(self):
    f, c = ctypes.c_double(), ctypes.c_double()
    n = REF().ref_de_params(self.h, ctypes.byref(f), ctypes.byref(c))
    return (f.value, c.value) if n else None


RefDE.params = _refde_params


def ref_param_record(series, problem_ids, instances, runs, dim=10):
    """The reference parameter_record fed with per-run [(generation, mu_f, mu_cr), ...] series."""
    n = max(1, max(len(s) for s in series))
    gens = np.zeros((len(series), n), np.int32)
    mf = np.zeros((len(series), n))
    mc = np.zeros((len(series), n))
    counts = np.array([len(s) for s in series], np.int32)
    for r, s in enumerate(series):
        for e, (g, a, b) in enumerate(s):
            gens[r, e], mf[r, e], mc[r, e] = g, a, b
    ids = np.ascontiguousarray(problem_ids, np.int32)
    args = (ptr(gens), ptr(mf), ptr(mc), n, ptr(counts), len(ids), ptr(ids), instances, runs, dim)
    ln = REF().ref_param_record(*args, None, 0)
    buf = ctypes.create_string_buffer(int(ln) + 1)
    REF().ref_param_record(*args, buf, int(ln))
    return buf.raw[:ln].decode()


register_c({"orc_cso_generation_f64": (i64, [c_int, c_int, c_double, c_int, vp, vp, c_double, vp, vp, vp, c_double,
                                             c_double, vp, i64])})


def cso_generation_c(P, D, phi, kind, shift, rot, bias, x, v, fit, lb, ub, words):
    """The C restatement of cso_optimizer::generation (in place on x, v, fit); returns words used."""
    o = np.ascontiguousarray(shift, np.float64)
    m = np.ascontiguousarray(rot, np.float64).ravel()
    w = np.ascontiguousarray(words, np.uint64)
    return int(C().orc_cso_generation_f64(P, D, phi, kind, ptr(o), ptr(m), bias, ptr(x), ptr(v), ptr(fit), lb, ub,
                                          ptr(w), len(w)))


register_ref({"ref_restart_lshade": (c_double, [ctypes.c_uint64, ctypes.c_uint64, c_int, c_int, c_int, c_double,
                                                 c_double, c_int, ctypes.c_longlong, ctypes.c_longlong, c_double,
                                                 c_int, vp, vp, c_double, vp, vp, c_double, c_double])})


def ref_restart_lshade(seed, stream, P, D, H, p_best, archive_rate, n_min, budget, stagnation, eps, kind, shift, rot,
                       bias=0.0, lb=-100.0, ub=100.0):
    o = np.ascontiguousarray(shift, np.float64)
    m = np.ascontiguousarray(rot, np.float64).ravel()
    runs, ev = ctypes.c_int(), ctypes.c_longlong()
    best = REF().ref_restart_lshade(seed, stream, P, D, H, p_best, archive_rate, n_min, budget, stagnation, eps, kind,
                                    ptr(o), ptr(m), bias, ctypes.byref(runs), ctypes.byref(ev), lb, ub)
    return {"best_fitness": best, "engine_runs": runs.value, "evaluations": ev.value}
