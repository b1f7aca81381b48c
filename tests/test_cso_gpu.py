"""GPU parity of the Competitive Swarm Optimizer (csrc/cso.cu) against the UNMODIFIED reference
cso_optimizer<T> (pso/cso.hpp, oracle/_ref): the device generation is the reference's generation
(data-parallel by construction), so positions, velocities and fitness must agree bit for bit on
transcendental-free objectives, generation after generation, in fp64 and fp32; and optimize() on
the reference's native stream (WORDS mode) must find the reference's best."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.cso import CSOEngine, scripted_words_for_generation  # noqa: E402
from paper_2505_17430_b200.de import Rng  # noqa: E402
from paper_2505_17430_b200.recorder import BestSoFarRecorder  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

K = evb.BaseKind


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("kind,P,D", [(K.elliptic, 64, 20), (K.sphere, 200, 100), (K.elliptic, 1024, 1000)])
def test_cso_generations_match_reference(dev, dtype, kind, P, D):
    nd = np.float64 if dtype == "f64" else np.float32
    tdt = torch.float64 if dtype == "f64" else torch.float32
    edt = evb.EVB_F64 if dtype == "f64" else evb.EVB_F32
    key, G, phi = 0xC50 + P, 6, 0.1
    o, m = O.shift_rotation(41, D)
    prob = evb.ProblemInstance.base(kind, o.astype(nd), m.astype(nd), 0.0, dtype=edt)
    rs = np.random.default_rng(P + D)
    x0 = rs.uniform(-100, 100, (P, D)).astype(nd)
    v0 = rs.uniform(-5, 5, (P, D)).astype(nd)
    X = torch.from_numpy(x0.copy()).to(dev)
    V = torch.from_numpy(v0.copy()).to(dev)
    fit = torch.empty(P, dtype=tdt, device=dev)
    evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
    ref = O.RefCSO(phi, P, D, int(kind), o.astype(nd), m.astype(nd), 0.0, dtype=nd)
    ref.set(x0, v0, fit.cpu().numpy())
    eng = CSOEngine(phi, P, D, dtype=edt)
    rng = Rng.philox(key)
    for g in range(G):
        eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
        assert ref.step(scripted_words_for_generation(key, g, P, D, philox=O.philox_words), -100.0, 100.0), g
        st = ref.get()
        assert np.array_equal(X.cpu().numpy(), st["x"]), g
        assert np.array_equal(V.cpu().numpy(), st["v"]), g
        if D < 200 or dtype == "f64":
            # large-D batched evaluation accumulates in a different order: compare within 1e-10 / 1e-4
            got = fit.cpu().numpy()
            tol = 1e-10 if dtype == "f64" else 1e-4
            assert np.all(np.abs(got - st["fit"]) <= tol * np.maximum(1, np.abs(st["fit"]))), g


def test_cso_optimize_native_stream(dev):
    # WORDS mode on rng_stream(seed, 0): the reference's own optimize() on its native stream
    P, D, max_fes, seed = 40, 10, 40 + 20 * 30, 77
    o, m = O.shift_rotation(seed, D)
    prob = evb.ProblemInstance.base(K.sphere, o, m, 0.0)
    n_words = P * D + 30 * ((P - 1) + (P // 2) * 3 * D)
    rng = Rng.words(O.rng_words(seed, 0, n_words))
    eng = CSOEngine(0.1, P, D)
    X = torch.empty((P, D), dtype=torch.float64, device=dev)
    V = torch.empty((P, D), dtype=torch.float64, device=dev)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    rec = BestSoFarRecorder(1, max_fes, 20)
    eng.attach_recorder(rec, 0)
    res = eng.optimize(prob, X, V, fit, -100.0, 100.0, max_fes, rng)
    rec.finish()
    assert res["generations"] == 30
    assert rng.state()["cursor"] == n_words and not rng.state()["overflow"]
    ref = O.RefCSO(0.1, P, D, int(K.sphere), o, m, 0.0)
    best = ref.native_optimize(seed, 0, -100.0, 100.0, max_fes)
    assert res["best_fitness"] == best
    grid, fes = rec.grid()
    assert fes[0] == max_fes and grid[0, -1] == best


def test_cso_errors(dev):
    with pytest.raises(evb.ConfigError):
        CSOEngine(0.1, 7, 3)
    with pytest.raises(evb.ConfigError):
        CSOEngine(-1.0, 8, 3)
    with pytest.raises(evb.ConfigError):
        CSOEngine(float("nan"), 8, 3)
