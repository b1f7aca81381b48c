"""GPU parity of the device best-so-far recorder (csrc/recorder.cu) against the reference's
experiment::best_so_far_record (experiment/recorder.hpp:35-155, driven through oracle/_ref's
ref_record): the checkpoint grid bit for bit and the CSV byte for byte, on raw value sequences
(ties, NaN, early-stopping runs, partial last interval) and on the FE sequences that the DE
engine and the batched-runs kernel report while they run."""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de  # noqa: E402
from paper_2505_17430_b200.recorder import BestSoFarRecorder  # noqa: E402
from paper_2505_17430_b200.runs import de_runs, run_keys  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")]


def same_grid(a, b):
    return np.array_equal(a, b, equal_nan=True)


def close_grid(a, b, tol):
    return a.shape == b.shape and bool(np.all(np.abs(a - b) <= tol * np.maximum(1.0, np.abs(b))))


def csv_close(a, b, tol):
    ra, rb = a.splitlines(), b.splitlines()
    if len(ra) != len(rb) or ra[0] != rb[0] or not a.endswith("\n"):
        return False
    for x, y in zip(ra[1:], rb[1:]):
        fx, fy = x.split(","), y.split(",")
        if fx[:-1] != fy[:-1] or abs(float(fx[-1]) - float(fy[-1])) > tol * max(1.0, abs(float(fy[-1]))):
            return False
    return True


@pytest.mark.parametrize("max_fes,interval", [(1000, 100), (1000, 7), (999, 1000 // 3), (50, 50)])
def test_raw_sequences_match_reference(dev, max_fes, interval):
    rs = np.random.default_rng(max_fes + interval)
    runs = 6
    seqs = []
    for r in range(runs):
        n = [max_fes, max_fes // 2, 3, 0, max_fes + 37, interval - 1][r]  # full, early stop, overrun
        v = np.round(rs.standard_normal(n) * 1e3, 1)  # rounding makes ties
        if n > 5:
            v[rs.integers(0, n, 3)] = np.nan
            v[0] = np.nan if r == 1 else v[0]
        seqs.append(v)
    ref_grid, ref_csv = O.ref_record(seqs, 10, max_fes, interval)
    rec = BestSoFarRecorder(runs, max_fes, interval)
    for r, v in enumerate(seqs):
        if len(v):
            # split into uneven chunks: observe is incremental across calls
            cuts = sorted(set([0, len(v)] + list(rs.integers(0, len(v), 3))))
            for a, b in zip(cuts[:-1], cuts[1:]):
                rec.observe(r, torch.from_numpy(v[a:b].copy()).to(dev))
    rec.finish()
    grid, fes = rec.grid()
    assert same_grid(grid, ref_grid)
    assert list(fes) == [len(v) for v in seqs]
    assert rec.to_csv("gpu", 10, [1], 1, runs) == ref_csv


def test_csv_layout_problems_instances(dev):
    # run index = (problem * instances + instance) * runs + run, as recorder.hpp:103-121 orders rows
    rec = BestSoFarRecorder(2 * 3 * 2, 40, 10)
    for r in range(12):
        rec.observe(r, torch.arange(40, 0, -1, dtype=torch.float64, device=dev) * (r + 1))
    rec.finish()
    csv = rec.to_csv("cec", 30, [4, 9], 3, 2).splitlines()
    assert csv[0] == "suite,problem,instance,dim,run,fes,best_so_far"
    assert len(csv) == 1 + 12 * 4
    assert csv[1] == "cec,4,1,30,1,10,31"
    assert csv[-1] == "cec,9,3,30,2,40,12"


@pytest.mark.parametrize("interval", [50, 64, 2100])
def test_de_engine_recording_matches_reference(dev, interval):
    # config-0 problem on the reference's native stream rng_stream(42, 0): the engine reports the
    # P initial evaluations and every generation's P trials in FE order; the reference engine's
    # objective-call trace fed to its own best_so_far_record must give the same grid and CSV
    P, D, G = 100, 10, 20
    o, m = O.shift_rotation(42, D)
    m = m * 0.0512
    cfg = preset_de(0.5, 0.9)
    prob = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m, 0.0)
    max_fes = P * (G + 1)
    words = O.rng_words(42, 0, P * D + G * P * (D + 40))
    rec = BestSoFarRecorder(1, max_fes, interval)
    eng = DEEngine(cfg, P, D)
    eng.attach_recorder(rec, 0)
    pop = torch.empty((P, D), dtype=torch.float64, device=dev)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    res = eng.optimize(prob, pop, fit, -100.0, 100.0, max_fes, Rng.words(words))
    rec.finish()
    assert res["generations"] == G
    ref = O.RefDE(cfg, P, D)
    ref.set_problem_base(5, o, m, 0.0)
    trace = ref.native_trace(42, 0, G, -100.0, 100.0)
    ref_grid, ref_csv = O.ref_record([trace], D, max_fes, interval)
    grid, fes = rec.grid()
    assert fes[0] == max_fes
    # populations are bit-exact (test_de_gpu); fitness values agree to 1e-12 (CUDA vs libm cos),
    # so the recorded minima do too and the CSV rows match field by field
    assert close_grid(grid, ref_grid, 1e-12)
    assert csv_close(rec.to_csv("gpu", D, [1], 1, 1), ref_csv, 1e-12)
    assert grid[0, -1] == fit.min().item()


def test_graph_replay_detached_recorder(dev):
    # attaching drops the cached graph (it does not contain the recorder call); later eager
    # generations keep recording, and detaching stops it
    P, D = 64, 20
    o, m = O.shift_rotation(5, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.ackley, o, m, 0.0)
    eng = DEEngine(preset_de(0.5, 0.9), P, D)
    rng = Rng.philox(5)
    pop = torch.empty((P, D), dtype=torch.float64, device=dev)
    eng.init_population(pop, -32.0, 32.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    eng.generations(prob, pop, fit, -32.0, 32.0, rng, 4)  # graph captured, no recorder
    rec = BestSoFarRecorder(1, 10 * P, P)
    eng.attach_recorder(rec, 0)
    eng.generations(prob, pop, fit, -32.0, 32.0, rng, 6)
    eng.attach_recorder(None)
    eng.generations(prob, pop, fit, -32.0, 32.0, rng, 3)
    grid, fes = rec.grid()
    assert fes[0] == 6 * P
    assert np.all(np.diff(grid[0, :6]) <= 0) and np.isnan(grid[0, 6:]).all()


def test_batched_runs_recording(dev):
    # K8 reports init + every generation's trials per run; the reference engine replays run 0's
    # Philox words and its objective trace through best_so_far_record
    from test_runs_gpu import D as D8, P as P8, make_runs
    n_runs, gens, interval = 6, 40, 250
    probs, comps = make_runs(n_runs)
    keys = run_keys(64, n_runs)
    pops = torch.empty((n_runs, P8, D8), dtype=torch.float64, device=dev)
    fits = torch.empty((n_runs, P8), dtype=torch.float64, device=dev)
    max_fes = P8 * (gens + 1)
    rec = BestSoFarRecorder(n_runs, max_fes, interval)
    de_runs(preset_de(0.5, 0.9), probs, keys, pops, fits, gens, -100.0, 100.0, init=True, gen0=0, recorder=rec)
    rec.finish()
    grid, fes = rec.grid()
    assert list(fes) == [max_fes] * n_runs
    f = fits.cpu().numpy()
    for r in range(n_runs):
        assert np.all(np.diff(grid[r]) <= 0)
        assert grid[r, -1] == f[r].min()
    s, mm = comps[0]
    ref = O.RefDE(preset_de(0.5, 0.9), P8, D8)
    ref.set_problem_composition(O.CONFIG4_KINDS, s, mm, O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA, O.CONFIG4_BIAS, 0.0)
    init_words = O.philox_words(int(keys[0]), (0 << 32) | 0xFFFFFFF0, 0, P8 * D8)
    assert ref.init(init_words, -100.0, 100.0) == P8 * D8
    trace = [ref.get()["fit"].copy()]
    for g in range(1, gens + 1):
        ok, vals = ref.generation_trace(O.de_fixed_generation_words(0, int(keys[0]), g, P8, D8), -100.0, 100.0)
        assert ok
        trace.append(vals)
    trace = np.concatenate(trace)
    ref_grid, _ = O.ref_record([trace], D8, max_fes, interval)
    # exact-order arithmetic: identical unless a libm-vs-CUDA ulp flipped a near-tie selection
    rel = np.abs(grid[0] - ref_grid[0]) / np.maximum(1.0, np.abs(ref_grid[0]))
    assert rel.max() <= 1e-10


def test_param_trace_shade_matches_reference(dev):
    # parameter_record (experiment/parameter_record.hpp): after every SHADE generation the engine
    # appends (generation, mean M_F, mean M_CR); compared with the reference adapter's own
    # append_parameters in lockstep, and the CSV with the reference parameter_record's
    from paper_2505_17430_b200.de import preset_shade, scripted_words_for_generation
    from paper_2505_17430_b200.recorder import ParamTrace
    P, D, G, key = 40, 12, 8, 0xAB
    o, m = O.shift_rotation(19, D)
    cfg = preset_shade(0.11, 10, 1.0)
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
    eng = DEEngine(cfg, P, D)
    trace = ParamTrace(1, 64)
    eng.attach_param_trace(trace, 0)
    rng = Rng.philox(key)
    pop = torch.empty((P, D), dtype=torch.float64, device=dev)
    eng.init_population(pop, -100.0, 100.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    ref = O.RefDE(cfg, P, D)
    ref.set_problem_base(0, o, m, 0.0)
    ref.set_pop(pop.cpu().numpy(), fit.cpu().numpy())
    for g in range(G):
        eng.generation(prob, pop, fit, -100.0, 100.0, rng)
        dr = eng.last_draws()
        assert ref.generation(scripted_words_for_generation(key, dr["generation"], dr["word_counts"],
                                                            dr["archive_words"], philox=O.philox_words),
                              -100.0, 100.0)
        gens, mf, mc = trace.series(0)
        assert list(gens) == list(range(1, g + 2))
        want = ref.params()
        assert abs(mf[-1] - want[0]) <= 1e-12 and abs(mc[-1] - want[1]) <= 1e-12, g
        st = ref.get()  # re-sync (F/CR ulps, as in the config-2 lockstep)
        pop.copy_(torch.from_numpy(st["pop"]))
        fit.copy_(torch.from_numpy(st["fit"]))
        eng.set_state(st["archive"], st["memory_f"], st["memory_cr"], st["write_index"])
    gens, mf, mc = trace.series(0)
    ref_csv = O.ref_param_record([list(zip(gens, mf, mc))], [3], 1, 1)
    assert trace.to_csv([3], 1, 1) == ref_csv


def test_param_trace_fixed_adapter_reports_nothing(dev):
    from paper_2505_17430_b200.recorder import ParamTrace
    P, D = 20, 5
    o, m = O.shift_rotation(3, D)
    prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
    eng = DEEngine(preset_de(), P, D)
    trace = ParamTrace(1, 8)
    eng.attach_param_trace(trace, 0)
    pop = torch.empty((P, D), dtype=torch.float64, device=dev)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    eng.optimize(prob, pop, fit, -100.0, 100.0, P * 5, Rng.philox(1))
    assert len(trace.series(0)[0]) == 0
    assert trace.to_csv([1], 1, 1) == "problem,instance,run,generation,mu_f,mu_cr\n"
