"""GPU parity of the synchronous PSO generation (K7) against the driver built from the reference's
own pieces (oracle/_ref), BASELINE config 3: w 0.7298, c1 = c2 = 1.49618, |v| <= 40, elliptic,
x ~ U[-100,100], v ~ U[-20,20], gbest and ring, fp64 and fp32.  Draws: Philox sub-streams,
replayed to the reference in its per-particle order."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import Rng  # noqa: E402
from paper_2505_17430_b200.pso import PSOEngine, config3, scripted_words_for_generation  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def run(dev, topology, nd, P, D, G, key=0xC0FFEE, lockstep=False):
    """G synchronous generations on the GPU and in the reference driver, compared after each.
    Positions and velocities must be bit-identical (same arithmetic, same draws).  A personal-best
    decision (strict <, pso/engine.hpp:78-79) may differ only at a flagged near-tie, where the two
    fitness values are within the tolerance (1e-10 fp64 / 1e-4 fp32 relative); the GPU's personal
    bests are then re-synced.  lockstep=True re-syncs them every generation (the GPU keeps its own
    evaluation of unchanged bests otherwise, and gbest / ring minima would see fp32 evaluation
    noise between near-equal particles).  Returns (worst relative fitness error, flagged)."""
    import os

    dtype = evb.EVB_F64 if nd == np.float64 else evb.EVB_F32
    tdt = torch.float64 if nd == np.float64 else torch.float32
    tol = 1e-10 if nd == np.float64 else 1e-4
    o, m = O.shift_rotation(13, D)
    o, m = o.astype(nd), m.astype(nd)
    prob = evb.ProblemInstance.base(evb.BaseKind.elliptic, o, m, 0.0, dtype=dtype)
    eng = PSOEngine(config3(topology), P, D, dtype)
    rng = Rng.philox(key)
    X = torch.empty((P, D), dtype=tdt, device=dev)
    V = torch.empty((P, D), dtype=tdt, device=dev)
    eng.init_uniform(X, -100.0, 100.0, rng)
    eng.init_uniform(V, -20.0, 20.0, rng)
    fit = torch.empty(P, dtype=tdt, device=dev)
    evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
    eng.prepare(X, fit)
    ref = O.RefPSO(nd, 0 if topology == "gbest" else 1, 0.7298, 1.49618, 1.49618, 40.0, P, D, 1, o, m)
    ref.set_threads(os.cpu_count() or 1)
    ref.set(X.cpu().numpy(), V.cpu().numpy(), fit.cpu().numpy())
    worst, flagged = 0.0, 0
    for g in range(G):
        eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
        st_gpu = eng.personal_bests()
        words = scripted_words_for_generation(key, st_gpu["generation"], P, D, philox=O.philox_words)
        assert ref.step(words, -100.0, 100.0)
        st = ref.get()
        # positions / velocities: same arithmetic, same draws -> identical
        assert np.array_equal(X.cpu().numpy(), st["x"]), g
        assert np.array_equal(V.cpu().numpy(), st["v"]), g
        f = fit.cpu().numpy().astype(np.float64)
        rf = st["fit"].astype(np.float64)
        rel = np.max(np.abs(f - rf) / np.maximum(1.0, np.abs(rf)))
        worst = max(worst, rel)
        assert rel <= tol, g
        # pbest decisions (strict <) agree except where the two fitness values are within tolerance
        same = np.all(st_gpu["pbest"] == st["pbest"], axis=1)
        if not same.all():
            for i in np.where(~same)[0]:
                pf = float(st["pbest_fit"][i])
                assert abs(f[i] - pf) <= tol * max(1.0, abs(pf)), (g, i)
            flagged += int((~same).sum())
        if lockstep or not same.all():
            eng.set_personal_bests(st["pbest"], st["pbest_fit"])
    return worst, flagged


@pytest.mark.parametrize("topology", ["gbest", "lbest_ring"])
@pytest.mark.parametrize("nd", [np.float64, np.float32])
def test_config3_small(dev, topology, nd):
    run(dev, topology, nd, 64, 200, 6)


@pytest.mark.parametrize("topology", ["gbest", "lbest_ring"])
@pytest.mark.parametrize("nan_at", [[0], [3], [0, 7], [5, 6, 40], list(range(50))])
def test_nan_personal_bests(dev, topology, nan_at):
    # NaN personal-best fitness: gbest follows the reference's sequential strict-< scan
    # (pso/topology.hpp:28-34: index 0 when its fitness is NaN, else the first minimum over the
    # non-NaN entries), the ring its three-candidate scan (:44-54); a NaN best never improves
    # (f < NaN is false).  Same draws -> positions and velocities identical to the reference driver.
    P, D, key = 50, 12, 0xBAD
    o, m = O.shift_rotation(13, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
    eng = PSOEngine(config3(topology), P, D, evb.EVB_F64)
    rng = Rng.philox(key)
    X = torch.empty((P, D), dtype=torch.float64, device=dev)
    V = torch.empty((P, D), dtype=torch.float64, device=dev)
    eng.init_uniform(X, -100.0, 100.0, rng)
    eng.init_uniform(V, -20.0, 20.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
    fit[nan_at] = float("nan")
    eng.prepare(X, fit)
    ref = O.RefPSO(np.float64, 0 if topology == "gbest" else 1, 0.7298, 1.49618, 1.49618, 40.0, P, D, 0, o, m)
    ref.set(X.cpu().numpy(), V.cpu().numpy(), fit.cpu().numpy())
    for g in range(4):
        eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
        st_gpu = eng.personal_bests()
        words = scripted_words_for_generation(key, st_gpu["generation"], P, D, philox=O.philox_words)
        assert ref.step(words, -100.0, 100.0)
        st = ref.get()
        assert np.array_equal(X.cpu().numpy(), st["x"]), g
        assert np.array_equal(V.cpu().numpy(), st["v"]), g
        assert np.array_equal(np.isnan(st_gpu["pbest_fit"]), np.isnan(st["pbest_fit"])), g
        assert np.array_equal(st_gpu["pbest"], st["pbest"]), g


@pytest.mark.parametrize("P", [1, 2, 33, 50])
def test_ring_small_and_ragged_swarms(dev, P):
    # ring neighbours from warp shuffles: swarms below / across a warp and not a multiple of 32
    # (warp edges, the wrap of the ring, lanes past the swarm), against the reference driver
    run(dev, "lbest_ring", np.float64, P, 12, 4)


@pytest.mark.parametrize("topology", ["gbest", "lbest_ring"])
@pytest.mark.parametrize("nd", [np.float64, np.float32], ids=["f64", "f32"])
def test_config3_full_size_lockstep(dev, topology, nd):
    # BASELINE config 3 at its full size (D=1000, pop 1024), fp64 and fp32, 50 lockstep iterations
    worst, flagged = run(dev, topology, nd, 1024, 1000, 50, lockstep=True)
    print(f"config 3 {topology} {np.dtype(nd).name}: 50 iterations, worst rel fitness {worst:.3e}, "
          f"{flagged} flagged pbest near-ties")


def test_config3_all_500_iterations(dev):
    # one variant for the config's full length: gbest, fp64, D=1000, pop 1024, 500 iterations
    worst, flagged = run(dev, "gbest", np.float64, 1024, 1000, 500, lockstep=True)
    print(f"config 3 gbest f64: 500 iterations, worst rel fitness {worst:.3e}, {flagged} flagged pbest near-ties")


@pytest.mark.parametrize("topology", ["lbest_ring", "gbest"])
@pytest.mark.parametrize("nd,P,D", [(np.float64, 64, 30), (np.float32, 64, 30), (np.float64, 256, 1000)])
def test_spso2011_spherical_lockstep(dev, topology, nd, P, D):
    # SPSO2011 rule (pso/update.hpp:81-114 spherical_update + sample_in_ball :24-43) in the
    # synchronous generation: the reference driver applies the UNMODIFIED spherical_update with the
    # exported words (2D + 1 per particle) and must consume exactly that many.  log/cos/pow come
    # from CUDA vs glibc, so positions agree to ulps (tolerance), and the GPU is re-synced each
    # generation; the neighbour-is-self case (G from x and p* only) is exercised by gbest's best
    from paper_2505_17430_b200.pso import PSOConfig
    dtype = evb.EVB_F64 if nd == np.float64 else evb.EVB_F32
    tdt = torch.float64 if nd == np.float64 else torch.float32
    key, G = 0x5B0 + D, 6
    cfg = PSOConfig(topology, "spherical")
    o, m = O.shift_rotation(31, D)
    o, m = o.astype(nd), m.astype(nd)
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0, dtype=dtype)
    eng = PSOEngine(cfg, P, D, dtype)
    rng = Rng.philox(key)
    X = torch.empty((P, D), dtype=tdt, device=dev)
    V = torch.empty((P, D), dtype=tdt, device=dev)
    eng.init_uniform(X, -100.0, 100.0, rng)
    eng.init_uniform(V, -20.0, 20.0, rng)
    fit = torch.empty(P, dtype=tdt, device=dev)
    evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
    eng.prepare(X, fit)
    ref = O.RefPSO(nd, 0 if topology == "gbest" else 1, cfg.inertia, cfg.cognitive, cfg.social, 0.0, P, D, 0, o, m,
                   update=1, attraction=cfg.attraction)
    ref.set(X.cpu().numpy(), V.cpu().numpy(), fit.cpu().numpy())
    tol = 1e-9 if nd == np.float64 else 2e-4
    for g in range(G):
        eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
        st_gpu = eng.personal_bests()
        words = scripted_words_for_generation(key, st_gpu["generation"], P, D, philox=O.philox_words,
                                              update="spherical")
        assert ref.step(words, -100.0, 100.0), g
        st = ref.get()
        for name, got in (("x", X), ("v", V)):
            a = got.cpu().numpy().astype(np.float64)
            b = st[name].astype(np.float64)
            scale = np.maximum(1.0, np.abs(b))
            assert np.max(np.abs(a - b) / scale) <= tol, (g, name)
        X.copy_(torch.from_numpy(st["x"]))
        V.copy_(torch.from_numpy(st["v"]))
        fit.copy_(torch.from_numpy(st["fit"]))
        eng.set_personal_bests(st["pbest"], st["pbest_fit"])
