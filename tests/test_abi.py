"""CPU tests of the C-ABI boundary: libevb.so loads, exports every symbol include/evb.h declares,
and rejects bad configurations with the mapped reference error types before touching a GPU."""
import ctypes

import numpy as np
import pytest

import paper_2505_17430_b200 as evb
from paper_2505_17430_b200 import _lib


def test_library_loads_and_exports_every_declared_symbol():
    L = _lib.lib()
    declared = _lib.declared_symbols()
    assert len(declared) >= 16
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    assert L.evb_abi_version() == 1


def test_error_mapping_without_gpu():
    L = _lib.lib()
    h = ctypes.c_void_p()
    z = np.zeros(4)
    # bad dtype -> config_error
    st = L.evb_problem_create_base(7, 2, 0, ctypes.c_void_p(z.ctypes.data), ctypes.c_void_p(z.ctypes.data), 0.0,
                                   ctypes.byref(h))
    assert st == _lib.EVB_ERR_CONFIG
    assert b"dtype" in L.evb_last_error()
    # unknown kind -> config_error
    st = L.evb_problem_create_base(1, 2, 42, ctypes.c_void_p(z.ctypes.data), ctypes.c_void_p(z.ctypes.data), 0.0,
                                   ctypes.byref(h))
    assert st == _lib.EVB_ERR_CONFIG
    # dim 0 -> config_error
    with pytest.raises(evb.ConfigError):
        evb.ProblemInstance.base(0, np.zeros(0), np.zeros(0))
    # null problem on evaluate -> config_error
    st = L.evb_evaluate_batch(None, None, None, 0, 0, None, None)
    assert st == _lib.EVB_ERR_CONFIG


def test_hybrid_validation():
    with pytest.raises(evb.ConfigError):
        evb.ProblemInstance.hybrid(np.zeros(4), np.eye(4), [0, 0], [2, 1], [0, 1, 2, 3])  # sizes sum != dim
    with pytest.raises(evb.ConfigError):
        evb.ProblemInstance.hybrid(np.zeros(4), np.eye(4), [0, 0], [2, 2], [0, 1, 1, 3])  # not a permutation


def test_composition_validation():
    with pytest.raises(evb.ConfigError):
        evb.ProblemInstance.composition([0] * 9, np.zeros((9, 2)), np.zeros((9, 2, 2)), [1] * 9, [1] * 9, [0] * 9)


def test_product_path_does_not_import_oracle():
    import pathlib

    pkg = pathlib.Path(evb.__file__).resolve().parent
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f
    for f in list(pkg.rglob("*.cu")) + list(pkg.rglob("*.cuh")):
        assert "evb_oracle" not in f.read_text(), f
