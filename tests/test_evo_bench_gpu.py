"""GPU parity of the suite-level grouped launch (csrc/evo_bench.cu) against the
reference's own experiment::evo_bench (experiment/runner.hpp:101-160) with its
best_so_far_record and de_engine::optimize (oracle/_ref ref_evo_bench_de): the same suite, the
`de` preset, each task replaying the words of the GPU task's positional Philox stream.  The CSV
(experiment/recorder.hpp:103-121) produced on the GPU must match the reference's row for row."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import preset_de, preset_shade  # noqa: E402
from paper_2505_17430_b200.experiment import evo_bench_de, task_key  # noqa: E402
from paper_2505_17430_b200.recorder import BestSoFarRecorder  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]

K = evb.BaseKind


def csv_close(a, b, tol):
    ra, rb = a.splitlines(), b.splitlines()
    assert len(ra) == len(rb) and ra[0] == rb[0] and a.endswith("\n")
    worst = 0.0
    for x, y in zip(ra[1:], rb[1:]):
        fx, fy = x.split(","), y.split(",")
        assert fx[:-1] == fy[:-1], (x, y)
        worst = max(worst, abs(float(fx[-1]) - float(fy[-1])) / max(1.0, abs(float(fy[-1]))))
    return worst <= tol


def make_suite(D, kinds, instances):
    suite, flat = [], []
    for p, kind in enumerate(kinds):
        row = []
        for i in range(instances):
            o, m = O.shift_rotation(500 + 10 * p + i, D)
            row.append(evb.ProblemInstance.base(kind, o, m, 0.0))
            flat.append((int(kind), o, m))
        suite.append(row)
    return suite, flat


@pytest.mark.parametrize("D,P,max_fes,interval", [(10, 20, 20 * 25 + 7, 50), (30, 24, 24 * 40, 96)])
def test_evo_bench_matches_reference(dev, D, P, max_fes, interval):
    kinds, ids, instances, runs, seed = [K.rastrigin, K.ackley], [5, 6], 2, 3, 99
    suite, flat = make_suite(D, kinds, instances)
    tasks = len(kinds) * instances * runs
    rec = BestSoFarRecorder(tasks, max_fes, interval)
    res = evo_bench_de(preset_de(0.5, 0.9), P, suite, runs, max_fes, master_seed=seed, recorder=rec)
    assert res["path"] == "batched"
    gpu_csv = rec.to_csv("gpu", D, ids, instances, runs)
    gens = max(0, -(-(max_fes - P) // P))
    words = [O.de_task_words(task_key(seed, t), P, D, gens) for t in range(tasks)]
    ref_csv, ref_best = O.ref_evo_bench_de(0.5, 0.9, P, D, ids, instances, runs, max_fes, interval,
                                           [k for k, _, _ in flat], np.stack([o for _, o, _ in flat]),
                                           np.stack([m for _, _, m in flat]), 0.0, words)
    # exact-order arithmetic; fitness differs from libm only in cos/exp ulps
    assert csv_close(gpu_csv, ref_csv, 1e-10)
    assert np.all(np.abs(res["best"] - ref_best) <= 1e-10 * np.maximum(1.0, np.abs(ref_best)))
    grid, fes = rec.grid()
    assert list(fes) == [P * (gens + 1)] * tasks
    # the last checkpoint is at (max_fes // interval) * interval FEs; trials past it can still improve
    if (max_fes // interval) * interval == P * (gens + 1):
        assert np.array_equal(grid[:, -1], res["best"])
    else:
        assert np.all(grid[:, -1] >= res["best"])


def test_batched_and_engine_paths_agree(dev):
    # the persistent kernel and the per-generation engine consume the same positional stream
    D, P, max_fes, interval, runs = 12, 16, 16 * 20, 32, 2
    suite, _ = make_suite(D, [K.ackley, K.rastrigin], 2)
    grids = []
    for force in (False, True):
        rec = BestSoFarRecorder(8, max_fes, interval)
        res = evo_bench_de(preset_de(0.5, 0.9), P, suite, runs, max_fes, master_seed=3, recorder=rec,
                           force_engine=force)
        assert res["path"] == ("engine" if force else "batched")
        grids.append((rec.grid()[0], res["best"]))
    (g0, b0), (g1, b1) = grids
    assert np.allclose(g0, g1, rtol=1e-12, atol=0) and np.allclose(b0, b1, rtol=1e-12, atol=0)


def test_engine_path_shade(dev):
    # configurations outside the persistent kernel (SHADE + archive) run per task on the engine
    D, P, max_fes, runs = 20, 30, 30 * 12, 2
    suite, _ = make_suite(D, [K.elliptic], 3)
    rec = BestSoFarRecorder(6, max_fes, 30)
    res = evo_bench_de(preset_shade(0.11, P, 1.0), P, suite, runs, max_fes, master_seed=5, recorder=rec)
    assert res["path"] == "engine"
    grid, fes = rec.grid()
    assert np.all(fes == max_fes)
    assert np.all(np.diff(grid, axis=1) <= 0)
    assert np.array_equal(grid[:, -1], res["best"])
    csv = rec.to_csv("cec", D, [2], 3, runs)
    assert csv.count("\n") == 1 + 6 * 12


def test_evo_bench_errors(dev):
    suite, _ = make_suite(10, [K.sphere], 1)
    with pytest.raises(evb.ConfigError):
        evo_bench_de(preset_de(), 20, suite, 0, 100)
    with pytest.raises(evb.ConfigError):
        evo_bench_de(preset_de(), 20, suite, 1, 0)
    with pytest.raises(evb.ConfigError):
        evo_bench_de(preset_de(), 3, suite, 1, 100)


def test_engine_path_lshade(dev):
    # L-SHADE through optimize(): the population shrinks on schedule; the FE count stops at the
    # first generation boundary at or past max_fes (de/engine.hpp:124, core/state.hpp:40)
    from paper_2505_17430_b200.de import preset_lshade
    D, P, max_fes, runs = 10, 40, 40 * 10, 2
    suite, _ = make_suite(D, [K.rastrigin], 2)
    rec = BestSoFarRecorder(4, max_fes, 40)
    res = evo_bench_de(preset_lshade(0.11, P, 1.0, n_min=4), P, suite, runs, max_fes, master_seed=8, recorder=rec)
    assert res["path"] == "engine"
    grid, fes = rec.grid()
    assert np.all(fes >= max_fes) and np.all(fes < max_fes + P)
    assert np.all(fes != P * (max_fes // P))  # sizes shrank, so the count is not a multiple of P
    assert np.all(np.diff(grid, axis=1) <= 0)


def test_evo_bench_cso_matches_reference(dev):
    # the `cso` preset over a suite: GPU generations are the reference's generations, so with a
    # transcendental-free objective the CSV must equal the reference harness's byte for byte
    from paper_2505_17430_b200.cso import scripted_words_for_generation as cso_words
    from paper_2505_17430_b200.experiment import evo_bench_cso
    D, P, runs, seed, interval = 12, 20, 2, 5, 30
    max_fes = P + 15 * (P // 2) + 3
    kinds, ids, instances = [K.sphere, K.elliptic], [1, 2], 2
    suite, flat = make_suite(D, kinds, instances)
    tasks = len(kinds) * instances * runs
    rec = BestSoFarRecorder(tasks, max_fes, interval)
    res = evo_bench_cso(0.1, P, suite, runs, max_fes, master_seed=seed, recorder=rec)
    gens = -(-(max_fes - P) // (P // 2))
    words = []
    for t in range(tasks):
        key = task_key(seed, t)
        words.append(np.concatenate([O.philox_words(key, 0xFFFFFFF0, 0, P * D)] +
                                    [cso_words(key, g, P, D, philox=O.philox_words) for g in range(1, gens + 1)]))
    ref_csv, ref_best = O.ref_evo_bench_cso(0.1, P, D, ids, instances, runs, max_fes, interval,
                                            [k for k, _, _ in flat], np.stack([o for _, o, _ in flat]),
                                            np.stack([m for _, _, m in flat]), 0.0, words)
    assert rec.to_csv("gpu", D, ids, instances, runs) == ref_csv
    assert np.array_equal(res["best"], ref_best)


def test_evo_bench_pso_presets(dev):
    # "pso" (gbest + standard) and "spso2011" (ring + spherical) over a suite: synchronous
    # generations; the harness contract — FE counts, monotone checkpoints, best ==
    # the final checkpoint when max_fes is a generation boundary — holds
    from paper_2505_17430_b200.experiment import evo_bench_pso
    from paper_2505_17430_b200.pso import PSOConfig, preset_spso2011
    D, P, runs = 10, 20, 2
    max_fes = P * 12
    suite, _ = make_suite(D, [K.rastrigin, K.sphere], 2)
    for cfg in (PSOConfig("gbest", "standard"), preset_spso2011()):
        rec = BestSoFarRecorder(8, max_fes, P)
        res = evo_bench_pso(cfg, P, suite, runs, max_fes, master_seed=9, recorder=rec)
        grid, fes = rec.grid()
        assert np.all(fes == max_fes)
        assert np.all(np.diff(grid, axis=1) <= 0)
        assert np.array_equal(grid[:, -1], res["best"])


def test_batched_runs_hybrid_and_mixed_suite(dev):
    # the persistent kernel runs hybrid problems too (permuted chunks, problems/instance.hpp:97-112):
    # a suite mixing base, hybrid and composition problems in ONE launch agrees with the
    # per-task engine path (same positional streams, both exact-order evaluation)
    D, P, max_fes, runs = 20, 24, 24 * 15, 2
    rs = np.random.default_rng(4)
    o, m = O.shift_rotation(61, D)
    perm = rs.permutation(D)
    hyb = evb.ProblemInstance.hybrid(o, m, [int(K.elliptic), int(K.rastrigin), int(K.ackley)], [6, 8, 6], perm, 100.0)
    base = evb.ProblemInstance.base(K.griewank, *O.shift_rotation(62, D), 0.0)
    s3, m3 = O.composition_components(77, D)
    comp = evb.ProblemInstance.composition(O.CONFIG4_KINDS, s3, m3, O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA, O.CONFIG4_BIAS,
                                           0.0)
    suite = [[hyb], [base], [comp]]
    out = []
    for force in (False, True):
        rec = BestSoFarRecorder(3 * runs, max_fes, P)
        res = evo_bench_de(preset_de(0.5, 0.9), P, suite, runs, max_fes, master_seed=21, recorder=rec,
                           force_engine=force)
        assert res["path"] == ("engine" if force else "batched")
        out.append((rec.grid()[0], res["best"]))
    (g0, b0), (g1, b1) = out
    assert np.allclose(g0, g1, rtol=1e-12, atol=0) and np.allclose(b0, b1, rtol=1e-12, atol=0)
