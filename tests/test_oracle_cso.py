"""CPU: the C restatement of cso_optimizer::generation (oracle/evb_oracle.c) pinned bit-for-bit to
the UNMODIFIED reference cso_optimizer (oracle/_ref), several generations on one word stream."""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@pytest.mark.parametrize("kind,P,D", [(0, 20, 5), (1, 64, 12), (5, 30, 8)])
def test_cso_restatement_matches_reference(kind, P, D):
    o, m = O.shift_rotation(31 + D, D)
    rs = np.random.default_rng(P)
    x = rs.uniform(-100, 100, (P, D))
    v = rs.uniform(-5, 5, (P, D))
    fit = O.eval_batch(kind, o, m, 0.0, x)
    ref = O.RefCSO(0.1, P, D, kind, o, m, 0.0)
    ref.set(x, v, fit)
    xc, vc, fc = x.copy(), v.copy(), fit.copy()
    for g in range(5):
        words = rs.integers(0, 2**64 - 1, size=(P - 1) + (P // 2) * 3 * D + 8, dtype=np.uint64, endpoint=True)
        used = O.cso_generation_c(P, D, 0.1, kind, o, m, 0.0, xc, vc, fc, -100.0, 100.0, words)
        assert used == (P - 1) + (P // 2) * 3 * D
        assert ref.step(words[:used], -100.0, 100.0), g
        st = ref.get()
        assert np.array_equal(st["x"], xc) and np.array_equal(st["v"], vc), g
        assert np.array_equal(st["fit"], fc), g
