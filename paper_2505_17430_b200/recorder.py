"""Device-resident best-so-far recorder (experiment/recorder.hpp:35-155: best_so_far_record) over
the C ABI — the harness boundary on the GPU.  Engines report every evaluation
in FE order (evb_de_attach_recorder, evb_de_runs(..., recorder)); to_csv reproduces the
reference's CSV byte for byte (shortest round-trip values)."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from ._lib import EVB_F64, check
from .problems import _stream_ptr

_REG = False


def _sigs():
    global _REG
    if _REG:
        return
    P = ctypes.POINTER
    vp, i64, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    _lib.register_signatures({
        "evb_recorder_create": (c_int, [c_int, c_int, i64, i64, P(vp)]),
        "evb_recorder_destroy": (c_int, [vp]),
        "evb_recorder_checkpoints": (c_int, [vp]),
        "evb_recorder_observe": (c_int, [vp, c_int, vp, i64, vp]),
        "evb_recorder_finish": (c_int, [vp, c_int, c_int, vp]),
        "evb_recorder_grid": (c_int, [vp, vp, vp]),
        "evb_recorder_csv": (c_int, [vp, ctypes.c_char_p, c_int, c_int, vp, c_int, c_int, vp, i64, P(i64)]),
        "evb_de_attach_recorder": (c_int, [vp, vp, c_int]),
        "evb_param_trace_create": (c_int, [c_int, c_int, c_int, P(vp)]),
        "evb_param_trace_destroy": (c_int, [vp]),
        "evb_param_trace_get": (c_int, [vp, c_int, vp, vp, vp, c_int, P(c_int)]),
        "evb_param_trace_csv": (c_int, [vp, c_int, vp, c_int, c_int, vp, i64, P(i64)]),
        "evb_de_attach_param_trace": (c_int, [vp, vp, c_int]),
    })
    _lib.lib()
    _REG = True


class BestSoFarRecorder:
    def __init__(self, n_runs: int, max_fes: int, interval: int, dtype: int = EVB_F64):
        _sigs()
        self.n_runs, self.max_fes, self.interval, self.dtype = n_runs, max_fes, interval, dtype
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_recorder_create(dtype, n_runs, max_fes, interval, ctypes.byref(self._h)),
              "evb_recorder_create")
        self.checkpoints = int(_lib.lib().evb_recorder_checkpoints(self._h))

    @property
    def handle(self):
        return self._h

    def observe(self, run: int, values, stream=None) -> None:
        """on_evaluate for every value of a device tensor, in order."""
        check(_lib.lib().evb_recorder_observe(self._h, run, ctypes.c_void_p(values.data_ptr()), values.numel(),
                                              _stream_ptr(stream)), "recorder_observe")

    def finish(self, run0: int = 0, n: int | None = None, stream=None) -> None:
        """on_run_end for runs [run0, run0 + n)."""
        n = self.n_runs - run0 if n is None else n
        check(_lib.lib().evb_recorder_finish(self._h, run0, n, _stream_ptr(stream)), "recorder_finish")

    def grid(self):
        nd = np.float64 if self.dtype == EVB_F64 else np.float32
        g = np.zeros((self.n_runs, self.checkpoints), nd)
        f = np.zeros(self.n_runs, np.int64)
        check(_lib.lib().evb_recorder_grid(self._h, ctypes.c_void_p(g.ctypes.data), ctypes.c_void_p(f.ctypes.data)),
              "recorder_grid")
        return g, f

    def to_csv(self, suite: str, dim: int, problem_ids, instances: int, runs: int) -> str:
        ids = (ctypes.c_int * len(problem_ids))(*problem_ids)
        n = ctypes.c_int64()
        L = _lib.lib()
        check(L.evb_recorder_csv(self._h, suite.encode(), dim, len(problem_ids), ids, instances, runs, None, 0,
                                 ctypes.byref(n)), "recorder_csv")
        buf = ctypes.create_string_buffer(n.value + 1)
        check(L.evb_recorder_csv(self._h, suite.encode(), dim, len(problem_ids), ids, instances, runs, buf, n.value,
                                 ctypes.byref(n)), "recorder_csv")
        return buf.raw[:n.value].decode()

    def close(self):
        if self._h:
            _lib.lib().evb_recorder_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ParamTrace:
    """Device parameter_record (experiment/parameter_record.hpp:15-95): per run the (generation,
    mu_F, mu_CR) series an adaptive DE engine reports after each generation."""

    def __init__(self, n_runs: int, capacity: int = 1024, dtype: int = EVB_F64):
        _sigs()
        self.n_runs, self.capacity, self.dtype = n_runs, capacity, dtype
        self._h = ctypes.c_void_p()
        check(_lib.lib().evb_param_trace_create(dtype, n_runs, capacity, ctypes.byref(self._h)), "param_trace_create")

    @property
    def handle(self):
        return self._h

    def series(self, run: int):
        nd = np.float64 if self.dtype == EVB_F64 else np.float32
        g = np.zeros(self.capacity, np.int32)
        f = np.zeros(self.capacity, nd)
        c = np.zeros(self.capacity, nd)
        n = ctypes.c_int()
        check(_lib.lib().evb_param_trace_get(self._h, run, ctypes.c_void_p(g.ctypes.data), ctypes.c_void_p(f.ctypes.data),
                                             ctypes.c_void_p(c.ctypes.data), self.capacity, ctypes.byref(n)),
              "param_trace_get")
        m = min(n.value, self.capacity)
        return g[:m], f[:m], c[:m]

    def to_csv(self, problem_ids, instances: int, runs: int) -> str:
        ids = (ctypes.c_int * len(problem_ids))(*problem_ids)
        n = ctypes.c_int64()
        L = _lib.lib()
        check(L.evb_param_trace_csv(self._h, len(problem_ids), ids, instances, runs, None, 0, ctypes.byref(n)),
              "param_trace_csv")
        buf = ctypes.create_string_buffer(n.value + 1)
        check(L.evb_param_trace_csv(self._h, len(problem_ids), ids, instances, runs, buf, n.value, ctypes.byref(n)),
              "param_trace_csv")
        return buf.raw[:n.value].decode()

    def close(self):
        if self._h:
            _lib.lib().evb_param_trace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
