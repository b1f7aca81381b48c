"""Suite-level grouped launch (experiment/runner.hpp:101-160: evo_bench) for DE presets over the
C ABI: all (problem x instance x run) tasks at once, evaluations recorded on the device
(recorder.BestSoFarRecorder) so the reference's CSV comes from the GPU."""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import EVB_F64, check
from .de import DEConfig, _Cfg, _sigs as _de_sigs
from .pso import PSOConfig, _Cfg as _PsoCfg, _sigs as _pso_sigs
from .problems import ProblemInstance, _stream_ptr
from .recorder import _sigs as _rec_sigs

_REG = False


def _sigs():
    global _REG
    if _REG:
        return
    _de_sigs()
    _pso_sigs()
    _rec_sigs()
    vp, i64, c_int, c_double, u64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint64
    _lib.register_signatures({
        "evb_task_key": (u64, [u64, u64]),
        "evb_evo_bench_de": (c_int, [c_int, ctypes.POINTER(_Cfg), c_int, c_int, vp, c_int, c_int, c_int, i64, u64,
                                     c_double, c_double, vp, vp, vp, c_int, ctypes.POINTER(c_int), vp]),
        "evb_evo_bench_pso": (c_int, [c_int, ctypes.POINTER(_PsoCfg), c_int, c_int, vp, c_int, c_int, c_int, i64, u64,
                                      c_double, c_double, vp, vp, vp]),
        "evb_evo_bench_cso": (c_int, [c_int, c_double, c_int, c_int, vp, c_int, c_int, c_int, i64, u64, c_double,
                                      c_double, vp, vp, vp]),
    })
    _REG = True


def task_key(master_seed: int, task_index: int) -> int:
    _sigs()
    return int(_lib.lib().evb_task_key(master_seed, task_index))


def evo_bench_de(cfg: DEConfig, pop_size: int, suite: Sequence[Sequence[ProblemInstance]], runs: int, max_fes: int,
                 master_seed: int = 0, lb: float = -100.0, ub: float = 100.0, recorder=None, param_trace=None,
                 force_engine: bool = False, dtype: int = EVB_F64, stream=None):
    """evo_bench(make_algorithm(cfg, pop_size), suite, recorder, {runs, max_fes, master_seed}).
    suite[p][i] is instance i of problem p.  Returns {"best": per-task best fitness (task index
    ((p * instances) + i) * runs + r), "path": "batched" | "engine"}."""
    _sigs()
    flat = [inst for row in suite for inst in row]
    n_problems, instances = len(suite), len(suite[0])
    if any(len(row) != instances for row in suite):
        raise ValueError("evo_bench: every problem needs the same number of instances")
    dim = flat[0].dim
    handles = (ctypes.c_void_p * len(flat))(*[p.handle.value for p in flat])
    c = cfg.to_c()
    best = np.zeros(n_problems * instances * runs)
    path = ctypes.c_int()
    check(_lib.lib().evb_evo_bench_de(dtype, ctypes.byref(c), pop_size, dim, handles, n_problems, instances, runs,
                                      max_fes, master_seed, lb, ub, recorder.handle if recorder is not None else None,
                                      param_trace.handle if param_trace is not None else None,
                                      ctypes.c_void_p(best.ctypes.data), 1 if force_engine else 0, ctypes.byref(path),
                                      _stream_ptr(stream)), "evo_bench_de")
    return {"best": best, "path": "batched" if path.value == 1 else "engine"}


def _suite_args(suite, runs):
    flat = [inst for row in suite for inst in row]
    n_problems, instances = len(suite), len(suite[0])
    if any(len(row) != instances for row in suite):
        raise ValueError("evo_bench: every problem needs the same number of instances")
    handles = (ctypes.c_void_p * len(flat))(*[p.handle.value for p in flat])
    return flat[0].dim, handles, n_problems, instances, np.zeros(n_problems * instances * runs)


def evo_bench_pso(cfg: PSOConfig, pop_size: int, suite: Sequence[Sequence[ProblemInstance]], runs: int,
                  max_fes: int, master_seed: int = 0, lb: float = -100.0, ub: float = 100.0, recorder=None,
                  dtype: int = EVB_F64, stream=None):
    """evo_bench with the "pso" / "spso2011" presets (synchronous generation)."""
    _sigs()
    dim, handles, n_problems, instances, best = _suite_args(suite, runs)
    c = cfg.to_c()
    check(_lib.lib().evb_evo_bench_pso(dtype, ctypes.byref(c), pop_size, dim, handles, n_problems, instances, runs,
                                       max_fes, master_seed, lb, ub,
                                       recorder.handle if recorder is not None else None,
                                       ctypes.c_void_p(best.ctypes.data), _stream_ptr(stream)), "evo_bench_pso")
    return {"best": best}


def evo_bench_cso(phi: float, pop_size: int, suite: Sequence[Sequence[ProblemInstance]], runs: int, max_fes: int,
                  master_seed: int = 0, lb: float = -100.0, ub: float = 100.0, recorder=None, dtype: int = EVB_F64,
                  stream=None):
    """evo_bench with the "cso" preset (cso_optimizer(phi); the reference's generation exactly)."""
    _sigs()
    dim, handles, n_problems, instances, best = _suite_args(suite, runs)
    check(_lib.lib().evb_evo_bench_cso(dtype, phi, pop_size, dim, handles, n_problems, instances, runs, max_fes,
                                       master_seed, lb, ub, recorder.handle if recorder is not None else None,
                                       ctypes.c_void_p(best.ctypes.data), _stream_ptr(stream)), "evo_bench_cso")
    return {"best": best}
