"""CPU: the C restatement of the synchronous PSO generation pinned to the driver built from the
reference's own topology / standard_update / bound pieces (oracle/_ref), fp64 and fp32; plus the
reference KATs (tests/test_pso.cpp:37-68)."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("nd", [np.float64, np.float32])
@pytest.mark.parametrize("topology", [0, 1])
def test_c_pso_matches_reference_pieces(nd, topology):
    P, D, G = 24, 16, 5
    o, m = O.shift_rotation(13, D)
    o, m = o.astype(nd), m.astype(nd)
    rng = np.random.default_rng(topology)
    x = rng.uniform(-100, 100, (P, D)).astype(nd)
    v = rng.uniform(-20, 20, (P, D)).astype(nd)
    fit = O.eval_batch(1, o, m, 0.0, x).astype(nd) if nd == np.float64 else None
    if fit is None:
        fit = np.array([O.C().orc_eval_scalar_f32(1, D, O.ptr(o), O.ptr(np.ascontiguousarray(m)), 0.0,
                                                  O.ptr(np.ascontiguousarray(x[i]))) for i in range(P)], nd)
    ref = O.RefPSO(nd, topology, 0.7298, 1.49618, 1.49618, 40.0, P, D, 1, o, m)
    ref.set(x, v, fit)
    pb, pbf = x.copy(), fit.copy()
    for g in range(G):
        words = rng.integers(0, 2**64 - 1, size=2 * P * D, dtype=np.uint64, endpoint=True)
        O.pso_step_c(topology, 0.7298, 1.49618, 1.49618, 40.0, 1, o, m, 0.0, x, v, fit, pb, pbf, words, -100.0, 100.0)
        assert ref.step(words, -100.0, 100.0)
        st = ref.get()
        for k, a in (("x", x), ("v", v), ("fit", fit), ("pbest", pb), ("pbest_fit", pbf)):
            assert np.array_equal(st[k], a), (g, k)


def test_topology_kats():
    # tests/test_pso.cpp:37-54 through the C restatement's neighbour export (identity problem)
    P, D = 4, 1
    pbf = np.array([3.0, 1.0, 2.0, 0.0])
    pb = np.zeros((P, D))
    x = np.zeros((P, D))
    v = np.zeros((P, D))
    fit = np.zeros(P)
    words = np.zeros(2 * P * D, np.uint64)
    nb = O.pso_step_c(1, 0.5, 1.0, 1.0, 0.0, 0, np.zeros(1), np.eye(1), 0.0, x, v, fit, pb.copy(), pbf.copy(), words,
                      -10.0, 10.0)
    assert nb[0] == 3 and nb[2] == 3 and nb[1] == 1  # ring
    nb = O.pso_step_c(0, 0.5, 1.0, 1.0, 0.0, 0, np.zeros(1), np.eye(1), 0.0, x, v, fit, pb.copy(), pbf.copy(), words,
                      -10.0, 10.0)
    assert nb[0] == 3  # gbest
    tied = np.ones(4)
    nb = O.pso_step_c(1, 0.5, 1.0, 1.0, 0.0, 0, np.zeros(1), np.eye(1), 0.0, x, v, fit, pb.copy(), tied.copy(), words,
                      -10.0, 10.0)
    assert nb[2] == 1  # ties to the lowest index
    nb = O.pso_step_c(0, 0.5, 1.0, 1.0, 0.0, 0, np.zeros(1), np.eye(1), 0.0, x, v, fit, pb.copy(), tied.copy(), words,
                      -10.0, 10.0)
    assert nb[2] == 0


def test_standard_update_kat():
    # tests/test_pso.cpp:56-68: w 0.5, c1 = c2 = 1, x 0, p 2, l 4, v 1, r1 = r2 = 1 - 2^-53 -> 6.5
    near_one = ((1 << 53) - 1) << 11
    x = np.zeros((2, 1))
    v = np.array([[1.0], [0.0]])
    pb = np.array([[2.0], [4.0]])
    pbf = np.array([1.0, 0.0])  # particle 1 is the gbest: l = 4 for particle 0
    fit = np.zeros(2)
    words = np.array([near_one] * 4, np.uint64)
    O.pso_step_c(0, 0.5, 1.0, 1.0, 0.0, 0, np.zeros(1), np.eye(1), 0.0, x, v, fit, pb, pbf, words, -100.0, 100.0)
    assert v[0, 0] == pytest.approx(6.5, rel=1e-12)
