"""CPU tests: the C restatement (oracle/evb_oracle.c) pinned against the reference's own
known-answer tests and against golden vectors produced by the reference itself
(tests/golden/*.npz, oracle/make_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def test_rng_regression_fixture():
    # tests/test_rng.cpp:20-30
    assert int(O.rng_words(42, 0, 1)[0]) == 0xA4137633ECF9D55D
    assert int(O.rng_words(42, 1, 1)[0]) == 0x176EDED3ECA867E4


def test_rng_matches_reference_words():
    g = np.load(GOLD / "rng.npz")
    for key in g.files:
        _, seed, stream = key.split("_")
        assert np.array_equal(O.rng_words(int(seed), int(stream), 16), g[key]), key


def test_uniform_int_forcing():
    # tests/support/forcing.hpp:12-15: word ((k << 64) + 2^63) / n gives uniform_int(n) == k
    for n in (3, 4, 7, 100, 180, 360, 1000):
        for k in (0, 1, n // 2, n - 1):
            w = ((k << 64) + (1 << 63)) // n
            assert O.C().orc_uniform_int_word(w, n) == k


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32-10
    kats = [
        ([0, 0, 0, 0], [0, 0], [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]),
        ([0xFFFFFFFF] * 4, [0xFFFFFFFF] * 2, [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]),
        ([0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344], [0xA4093822, 0x299F31D0],
         [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]),
    ]
    for ctr, key, want in kats:
        c = np.array(ctr, np.uint32)
        k = np.array(key, np.uint32)
        o = np.empty(4, np.uint32)
        O.C().orc_philox_block(O.ptr(c), O.ptr(k), O.ptr(o))
        assert [int(v) for v in o] == want


def test_philox_word_layout():
    # word n = (out[2*(n&1)+1] << 32) | out[2*(n&1)] of block n >> 1
    key, hi = 0x0123456789ABCDEF, 5
    c = np.array([3, 0, hi, 0], np.uint32)
    k = np.array([key & 0xFFFFFFFF, key >> 32], np.uint32)
    o = np.empty(4, np.uint32)
    O.C().orc_philox_block(O.ptr(c), O.ptr(k), O.ptr(o))
    w = O.philox_words(key, hi, 6, 2)
    assert int(w[0]) == (int(o[1]) << 32) | int(o[0])
    assert int(w[1]) == (int(o[3]) << 32) | int(o[2])


def test_base_kernel_known_values():
    # tests/test_problems.cpp:39-59
    C = O.C()

    def val(kind, z):
        z = np.ascontiguousarray(z, np.float64)
        return C.orc_base_value_f64(kind, O.ptr(z), len(z))

    zeros = np.zeros(5)
    assert val(0, zeros) == 0.0
    assert val(5, zeros) == 0.0
    assert abs(val(6, zeros)) < 1e-12
    assert val(7, zeros) == 0.0
    assert val(8, zeros) == 0.0
    assert val(9, zeros) == 0.0
    assert val(0, [1.0, 2.0, 3.0]) == 14.0
    # rosenbrock is evaluated on z + 1 (base_value_origin): zero at z = 0
    assert val(4, np.zeros(7)) == 0.0
    assert val(1, [1.0, 1.0]) == pytest.approx(1.0 + 1e6)
    assert val(2, [1.0, 1.0]) == pytest.approx(1.0 + 1e6)
    assert val(3, [1.0, 1.0]) == pytest.approx(1.0 + 1e6)
    assert val(8, [1.0, 1.0]) == pytest.approx(5.0)


def test_transform_linear_algebra():
    # tests/test_problems.cpp:61-79 through the scalar path: identity and 90-degree rotation
    o = np.array([1.0, 2.0])
    eye = np.eye(2)
    assert O.eval_batch(0, o, eye, 0.0, np.array([[1.0, 2.0]]))[0] == 0.0
    assert O.eval_batch(0, o, eye, 0.0, np.array([[3.0, 5.0]]))[0] == 13.0
    rot = np.array([[0.0, -1.0], [1.0, 0.0]])
    assert O.eval_batch(0, o, rot, 0.0, np.array([[2.0, 2.0]]))[0] == pytest.approx(1.0)


def test_rotation_is_orthogonal():
    # tests/test_problems.cpp:99-121
    for dim in (10, 50):
        _, m = O.shift_rotation(123, dim)
        assert np.max(np.abs(m @ m.T - np.eye(dim))) < 1e-10


def test_shift_range():
    o, _ = O.shift_rotation(5, 100)
    assert np.all(o >= -80.0) and np.all(o <= 80.0)


@pytest.mark.parametrize("dim", [16, 50])
def test_eval_matches_reference_golden(dim):
    g = np.load(GOLD / "eval.npz")
    o, m, x = g[f"shift_{dim}"], g[f"rot_{dim}"], g[f"x_{dim}"]
    # the restated generators reproduce the reference's own draws
    o2, m2 = O.shift_rotation(7 + dim, dim)
    assert np.array_equal(o, o2) and np.array_equal(m, m2)
    assert np.array_equal(x, O.population(8 + dim, x.shape[0], dim))
    for kind in range(10):
        got = O.eval_batch(kind, o, m, 100.0, x)
        assert np.array_equal(got, g[f"f64_{dim}_{kind}"]), kind
        got32 = O.eval_batch(kind, o.astype(np.float32), m.astype(np.float32), 100.0, x.astype(np.float32))
        assert np.array_equal(got32, g[f"f32_{dim}_{kind}"]), kind
    got = O.eval_hybrid(o, m, 900.0, g[f"hyb_kinds_{dim}"], g[f"hyb_sizes_{dim}"], g[f"hyb_perm_{dim}"], x)
    assert np.array_equal(got, g[f"hyb_{dim}"])
    got = O.eval_composition([5, 1, 6], g[f"comp_shifts_{dim}"], g[f"comp_rots_{dim}"], [10.0, 20.0, 30.0],
                             [1.0, 1e-6, 1.0], [0.0, 100.0, 200.0], 0.0, g[f"comp_x_{dim}"])
    assert np.array_equal(got, g[f"comp_{dim}"])
    assert got[0] == pytest.approx(100.0)  # zero-distance collapse onto component 1


def test_composition_rules():
    # tests/test_problems.cpp:193-237 with identity rotations
    eye = np.eye(3)
    # at a component's shift that component dominates: lambda*f(0)+bias = 5
    got = O.eval_composition([0, 5], [[1, 1, 1], [-3, 0, 2]], [eye, eye], [10, 20], [2.0, 1.0], [5.0, 100.0], 0.0,
                             np.array([[1.0, 1.0, 1.0]]))
    assert got[0] == pytest.approx(5.0)
    # single component reduces to shifted base + bias
    got = O.eval_composition([0], [[1, 2, 3]], [eye], [10], [1.0], [7.0], 0.0, np.array([[2.0, 2.0, 2.0]]))
    assert got[0] == pytest.approx(9.0)
    # two identical components split evenly, also at the shared shift
    got = O.eval_composition([0, 0], [[1, 1, 1], [1, 1, 1]], [eye, eye], [10, 10], [1.0, 1.0], [0.0, 10.0], 0.0,
                             np.array([[4.0, 4.0, 4.0], [1.0, 1.0, 1.0]]))
    assert got[0] == pytest.approx(0.5 * 27 + 0.5 * 37)
    assert got[1] == pytest.approx(5.0)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_c_oracle_matches_reference_binary_random():
    R = O.REF()
    rng = np.random.default_rng(0)
    for dim in (1, 2, 3, 10, 33):
        o, m = O.shift_rotation(dim, dim)
        x = rng.uniform(-100, 100, size=(5, dim))
        mr = np.ascontiguousarray(m.ravel())
        for kind in range(10):
            ref = np.empty(5)
            R.ref_eval_batch_f64(kind, dim, O.ptr(o), O.ptr(mr), 3.0, 5, O.ptr(x), dim, O.ptr(ref))
            assert np.array_equal(O.eval_batch(kind, o, m, 3.0, x), ref), (dim, kind)
