"""Batched independent runs (K8) — the GPU analogue of the reference's evo_bench task pool
(experiment/runner.hpp:101-160) for DE runs of the `de` preset family: one persistent launch, one
CTA per run, every generation inside the kernel."""
from __future__ import annotations

import ctypes
from typing import Sequence

import numpy as np

from . import _lib
from ._lib import EVB_F64, check
from .de import DEConfig, _Cfg, _sigs as _de_sigs
from .problems import ProblemInstance, _stream_ptr

_REG = False


def _sigs():
    global _REG
    if _REG:
        return
    _de_sigs()
    vp, i64, c_int, c_double, u32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_uint32
    _lib.register_signatures({
        "evb_de_runs": (c_int, [c_int, ctypes.POINTER(_Cfg), c_int, c_int, c_int, vp, vp, c_int, c_double, c_double,
                                vp, vp, c_int, u32, vp, vp]),
    })
    _REG = True


def run_keys(master_seed: int, n_runs: int) -> np.ndarray:
    """Per-run Philox keys: splitmix64(master_seed ^ run) (the analogue of derive_stream(seed, task),
    experiment/runner.hpp:118-120)."""
    out = np.empty(n_runs, np.uint64)
    for r in range(n_runs):
        z = (master_seed ^ r) & 0xFFFFFFFFFFFFFFFF
        z = (z + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        out[r] = z ^ (z >> 31)
    return out


def de_runs(cfg: DEConfig, problems: Sequence[ProblemInstance], keys, pops, fits, generations: int, lb: float,
            ub: float, init: bool = True, gen0: int = 0, recorder=None, stream=None) -> None:
    """Run len(problems) independent DE runs for `generations` generations in one launch.
    pops: (n_runs, pop_size, dim) float64 CUDA tensor; fits: (n_runs, pop_size)."""
    _sigs()
    n_runs, P, D = pops.shape
    c = cfg.to_c()
    handles = (ctypes.c_void_p * n_runs)(*[p.handle.value for p in problems])
    k = np.ascontiguousarray(keys, np.uint64)
    check(_lib.lib().evb_de_runs(EVB_F64, ctypes.byref(c), n_runs, P, D, handles, ctypes.c_void_p(k.ctypes.data),
                                 generations, lb, ub, ctypes.c_void_p(pops.data_ptr()),
                                 ctypes.c_void_p(fits.data_ptr()), int(init), gen0,
                                 recorder.handle if recorder is not None else None, _stream_ptr(stream)), "de_runs")
