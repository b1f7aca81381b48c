"""GPU parity of batched evaluation (K1 fp64 / K2 fp32 / small-D / z-store / hybrid / composition)
against the C oracle (itself pinned to the reference, tests/test_oracle.py).

Tolerances (north_star): fitness within 1e-10 relative (fp64) and 1e-4 relative (fp32), with
the reference's own convention |d| <= tol * max(1, |ref|) (tests/test_problems.cpp:310, 328-329).
Small-D paths accumulate in the reference's exact order, so transcendental-free kinds are
required to be bit-identical there.
"""
import numpy as np
import pytest

import oracle as O

torch = pytest.importorskip("torch")
import paper_2505_17430_b200 as evb  # noqa: E402

pytestmark = pytest.mark.gpu

K = evb.BaseKind
ALL_KINDS = list(K)
NO_TRIG = [K.sphere, K.elliptic, K.bent_cigar, K.discus, K.rosenbrock, K.schwefel_12]


def rel_err(got, ref):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref)))) if ref.size else 0.0


def gpu_eval(problem, X, dev):
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
    out = torch.empty(X.shape[0], dtype=Xd.dtype, device=dev)
    evb.evaluate_batch(problem, Xd, sc, out)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.fixture(scope="module")
def config1():
    # BASELINE config 1: D=1000, pop=1024, seed 7 (SURVEY §8(d) stream assignment)
    o, m = O.shift_rotation(7, 1000)
    X = O.population(7, 1024, 1000)
    return o, m, X


@pytest.mark.parametrize("kind", [K.elliptic, K.rastrigin, K.ackley])
def test_config1_fp64(config1, dev, kind):
    o, m, X = config1
    p = evb.ProblemInstance.base(kind, o, m, 0.0)
    got = gpu_eval(p, X, dev)
    ref = O.eval_batch(int(kind), o, m, 0.0, X)
    assert rel_err(got, ref) <= 1e-10


@pytest.mark.parametrize("kind", [K.elliptic, K.rastrigin, K.ackley])
def test_config1_fp32(config1, dev, kind):
    o, m, X = config1
    o32, m32, X32 = o.astype(np.float32), m.astype(np.float32), X.astype(np.float32)
    p = evb.ProblemInstance.base(kind, o32, m32, 0.0, dtype=evb.EVB_F32)
    got = gpu_eval(p, X32, dev)
    ref = O.eval_batch(int(kind), o32, m32, 0.0, X32)
    assert rel_err(got, ref) <= 1e-4


def test_config1_three_on_one_z(config1, dev):
    o, m, X = config1
    kinds = [K.elliptic, K.rastrigin, K.ackley]
    p = evb.ProblemInstance.base(K.elliptic, o, m, 0.0)
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(X).to(dev)
    out = torch.empty((3, X.shape[0]), dtype=torch.float64, device=dev)
    evb.evaluate_batch_multi(p, kinds, [0.0, 100.0, 200.0], Xd, sc, out)
    got = out.cpu().numpy()
    for k, kind in enumerate(kinds):
        ref = O.eval_batch(int(kind), o, m, 100.0 * k, X)
        assert rel_err(got[k], ref) <= 1e-10, kind


@pytest.mark.parametrize("dtype", [evb.EVB_F64, evb.EVB_F32])
@pytest.mark.parametrize("kind", ALL_KINDS)
def test_all_kinds_large_dim(dev, kind, dtype):
    # D=1000 (1000-D parity of every base kind, tests/test_problems.cpp:370-401) with a ragged
    # batch; rosenbrock / schwefel / schaffer take the z-store + row path
    o, m = O.shift_rotation(64, 1000)
    X = O.population(65, 37, 1000)
    nd = np.float64 if dtype == evb.EVB_F64 else np.float32
    o, m, X = o.astype(nd), m.astype(nd), X.astype(nd)
    p = evb.ProblemInstance.base(kind, o, m, 100.0, dtype=dtype)
    got = gpu_eval(p, X, dev)
    ref = O.eval_batch(int(kind), o, m, 100.0, X)
    assert rel_err(got, ref) <= (1e-10 if dtype == evb.EVB_F64 else 1e-4)


@pytest.mark.parametrize("dim", [1, 2, 10, 30, 50, 100])
@pytest.mark.parametrize("dtype", [evb.EVB_F64, evb.EVB_F32])
def test_small_dim_exact_order(dev, dim, dtype):
    o, m = O.shift_rotation(3 + dim, dim)
    X = O.population(4 + dim, 13, dim)
    nd = np.float64 if dtype == evb.EVB_F64 else np.float32
    o, m, X = o.astype(nd), m.astype(nd), X.astype(nd)
    for kind in ALL_KINDS:
        p = evb.ProblemInstance.base(kind, o, m, 100.0 * (int(kind) + 1), dtype=dtype)
        got = gpu_eval(p, X, dev)
        ref = O.eval_batch(int(kind), o, m, 100.0 * (int(kind) + 1), X)
        if kind in NO_TRIG:
            assert np.array_equal(got, ref), (kind, dim)
        else:
            assert rel_err(got, ref) <= (1e-12 if dtype == evb.EVB_F64 else 1e-6), (kind, dim)


def test_evaluate_at_shift_is_bias(dev):
    # tests/test_problems.cpp:124-130
    for dim in (10, 1000):
        o, m = O.shift_rotation(99, dim)
        for kind in ALL_KINDS:
            p = evb.ProblemInstance.base(kind, o, m, 100.0 * (int(kind) + 1))
            got = gpu_eval(p, o.reshape(1, -1), dev)
            assert abs(got[0] - 100.0 * (int(kind) + 1)) <= 1e-10 * 100.0 * (int(kind) + 1), (kind, dim)


def test_identity_sphere_114(dev):
    # tests/test_problems.cpp:132-139: identity sphere at (1,2,3) with bias 100 is exactly 114
    p = evb.ProblemInstance.base(K.sphere, np.zeros(3), np.eye(3), 100.0)
    got = gpu_eval(p, np.array([[1.0, 2.0, 3.0]]), dev)
    assert got[0] == 114.0


@pytest.mark.parametrize("dim", [10, 100, 1000])
def test_hybrid(dev, dim):
    o, m = O.shift_rotation(11, dim)
    X = O.population(12, 21, dim)
    rng = np.random.default_rng(dim)
    perm = rng.permutation(dim).astype(np.int32)
    for kinds, props in (([K.schwefel_12, K.rastrigin, K.elliptic], [0.3, 0.3, 0.4]),
                         ([K.discus, K.griewank, K.rosenbrock, K.sphere], [0.2, 0.2, 0.3, 0.3])):
        sizes = []
        used = 0
        for c, pr in enumerate(props[:-1]):  # problems/instance.hpp:300-313
            s = int(np.ceil(pr * dim))
            s = max(1, min(s, dim - used - (len(props) - 1 - c)))
            sizes.append(s)
            used += s
        sizes.append(dim - used)
        p = evb.ProblemInstance.hybrid(o, m, [int(k) for k in kinds], sizes, perm, 900.0)
        got = gpu_eval(p, X, dev)
        ref = O.eval_hybrid(o, m, 900.0, [int(k) for k in kinds], sizes, perm, X)
        assert rel_err(got, ref) <= 1e-10


@pytest.mark.parametrize("dim", [10, 50, 200])
@pytest.mark.parametrize("dtype", [evb.EVB_F64, evb.EVB_F32])
def test_composition(dev, dim, dtype):
    # BASELINE config 4 composition: rastrigin / elliptic / ackley, sigma (10,20,30),
    # lambda (1, 1e-6, 1), bias (0, 100, 200)
    nd = np.float64 if dtype == evb.EVB_F64 else np.float32
    shifts, rots = [], []
    for c in range(3):
        o, m = O.shift_rotation(1000 + c, dim)
        shifts.append(o)
        rots.append(m)
    shifts = np.stack(shifts).astype(nd)
    rots = np.stack(rots).astype(nd)
    kinds = [int(K.rastrigin), int(K.elliptic), int(K.ackley)]
    sigma, lam, cb = [10.0, 20.0, 30.0], [1.0, 1e-6, 1.0], [0.0, 100.0, 200.0]
    X = O.population(5, 33, dim).astype(nd)
    X[0] = shifts[1]  # zero-distance collapse onto component 1 (problems/instance.hpp:135-149)
    p = evb.ProblemInstance.composition(kinds, shifts, rots, sigma, lam, cb, 0.0, dtype=dtype)
    got = gpu_eval(p, X, dev)
    ref = O.eval_composition(kinds, shifts, rots, sigma, lam, cb, 0.0, X)
    assert rel_err(got, ref) <= (1e-10 if dtype == evb.EVB_F64 else 1e-4)
    assert abs(float(got[0]) - 100.0) <= 1e-6  # lambda_1 * f(0) + bias_1


def test_edge_cases(dev):
    o, m = O.shift_rotation(21, 1000)
    p = evb.ProblemInstance.base(K.rastrigin, o, m, 0.0)
    sc = evb.EvalScratch()
    # empty batch gives empty output (tests/test_problems.cpp:289-292)
    X0 = torch.empty((0, 1000), dtype=torch.float64, device=dev)
    out0 = torch.empty(0, dtype=torch.float64, device=dev)
    evb.evaluate_batch(p, X0, sc, out0)
    # single point, odd row pitch (not TMA-legal -> re-pitched), padded rows
    X = O.population(22, 5, 1000)
    ref = O.eval_batch(int(K.rastrigin), o, m, 0.0, X)
    for pad in (0, 1, 3, 24):
        Xp = np.zeros((5, 1000 + pad))
        Xp[:, :1000] = X
        Xd = torch.from_numpy(Xp).to(dev)[:, :1000]
        out = torch.empty(5, dtype=torch.float64, device=dev)
        evb.evaluate_batch(p, Xd, sc, out)
        assert rel_err(out.cpu().numpy(), ref) <= 1e-10, pad
    got1 = gpu_eval(p, X[:1], dev)
    assert rel_err(got1, ref[:1]) <= 1e-10
    # dimension mismatch -> std::invalid_argument analogue
    with pytest.raises(evb.InvalidArgument):
        evb.evaluate_batch(p, torch.zeros((3, 999), dtype=torch.float64, device=dev), sc,
                           torch.empty(3, dtype=torch.float64, device=dev))


def test_deterministic(config1, dev):
    o, m, X = config1
    p = evb.ProblemInstance.base(K.ackley, o, m, 0.0)
    a = gpu_eval(p, X, dev)
    b = gpu_eval(p, X, dev)
    assert np.array_equal(a, b)


def test_host_path(config1):
    o, m, X = config1
    p = evb.ProblemInstance.base(K.elliptic, o, m, 200.0)
    got = evb.batched_evaluate(p, X[:100])
    ref = O.eval_batch(int(K.elliptic), o, m, 200.0, X[:100])
    assert rel_err(got, ref) <= 1e-10
    assert evb.batched_evaluate(p, np.zeros((0, 1000))).size == 0
    with pytest.raises(evb.InvalidArgument):
        evb.batched_evaluate(p, np.zeros((2, 7)))


@pytest.mark.parametrize("kind", [K.elliptic, K.rastrigin, K.ackley, K.sphere])
def test_host_path_overlapped_copy_bit_identical(config1, dev, kind):
    # the host entry point streams X in column chunks gated per chunk into the fused fp64 GEMM:
    # results must equal the device-resident path bit for bit, call after call (gate epochs)
    o, m, X = config1
    p = evb.ProblemInstance.base(kind, o, m, 10.0)
    # (the tile shape, hence the fixed partial-sum grouping, depends on P: compare like with like)
    want = {rows: gpu_eval(p, X[:rows], dev) for rows in (1024, 37, 64)}
    sc = evb.EvalScratch()
    for rows in (1024, 1024, 37, 1024):
        got = evb.batched_evaluate(p, X[:rows], sc)
        assert np.array_equal(got, want[rows])
    wide = np.zeros((64, 1003))
    wide[:, :1000] = X[:64]
    got = evb.batched_evaluate(p, wide[:, :1000], sc)
    assert np.array_equal(got, want[64])


SWEEP = [(159, 63), (160, 65), (161, 1), (161, 300), (255, 129), (256, 64), (257, 65), (1003, 7), (2049, 65)]


@pytest.mark.parametrize("dim,n", SWEEP)
@pytest.mark.parametrize("dtype", [evb.EVB_F64, evb.EVB_F32])
def test_shape_sweep_path_boundaries(dev, dim, n, dtype):
    # around the small-D / GEMM switch (D = 160), the tile edges (56 / 64 / 128 / 32-float K-slices)
    # and ragged batches: every path against the C restatement; multi-output fused epilogue too
    o, m = O.shift_rotation(900 + dim, dim)
    X = O.population(901 + dim, n, dim)
    nd = np.float64 if dtype == evb.EVB_F64 else np.float32
    o, m, X = o.astype(nd), m.astype(nd), X.astype(nd)
    tol = 1e-10 if dtype == evb.EVB_F64 else 1e-4
    kinds = [K.elliptic, K.rastrigin, K.ackley, K.griewank]
    for kind in kinds:
        p = evb.ProblemInstance.base(kind, o, m, 7.0, dtype=dtype)
        assert rel_err(gpu_eval(p, X, dev), O.eval_batch(int(kind), o, m, 7.0, X)) <= tol, (kind, dim, n)
    p = evb.ProblemInstance.base(K.sphere, o, m, 0.0, dtype=dtype)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
    out = torch.empty((3, n), dtype=Xd.dtype, device=dev)
    evb.evaluate_batch_multi(p, [int(K.elliptic), int(K.rastrigin), int(K.ackley)], [1.0, 2.0, 3.0], Xd,
                             evb.EvalScratch(), out)
    got = out.cpu().numpy()
    for r, (kind, b) in enumerate(((K.elliptic, 1.0), (K.rastrigin, 2.0), (K.ackley, 3.0))):
        assert rel_err(got[r], O.eval_batch(int(kind), o, m, b, X)) <= tol, ("multi", kind, dim, n)


def test_host_many_one_copy_equals_device(config1, dev):
    # several problems on one host population: one H2D copy, results identical to the device path
    o, m, X = config1
    kinds = [K.elliptic, K.rastrigin, K.ackley, K.griewank]
    probs = [evb.ProblemInstance.base(k, o, m, float(i)) for i, k in enumerate(kinds)]
    want = [gpu_eval(p, X, dev) for p in probs]
    sc = evb.EvalScratch()
    for _ in range(2):
        got = evb.batched_evaluate_many(probs, X, sc)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)
    small = [evb.ProblemInstance.base(k, *O.shift_rotation(5, 30), 0.0) for k in kinds]
    Xs = O.population(6, 17, 30)
    for p, g in zip(small, evb.batched_evaluate_many(small, Xs, sc)):
        assert np.array_equal(g, gpu_eval(p, Xs, dev))
    with pytest.raises(evb.InvalidArgument):
        evb.batched_evaluate_many([probs[0], small[0]], X, sc)


@pytest.mark.parametrize("n_prob", [2, 3])
def test_host_many_row_split_gates(config1, dev, n_prob):
    # two or three problems on one host population: one multi-problem launch whose first wave is
    # the first rows' tiles, fed by two gate groups (first-wave rows, then the rest) of column
    # chunks; bit-identical to the device path, call after call, at one- and two-wave sizes
    o, m, X = config1
    o2, m2 = O.shift_rotation(8, 1000)
    specs = [(K.elliptic, o, m, 1.0), (K.rastrigin, o2, m2, 2.0), (K.ackley, o, m2, 3.0)][:n_prob]
    probs = [evb.ProblemInstance.base(k, oo, mm, b) for k, oo, mm, b in specs]
    big = np.concatenate([X, O.population(77, 1000, 1000)])  # 2024 rows: 32 row tiles
    sc = evb.EvalScratch()
    for rows in (1024, 2024, 600, 1024, 37, 2024):
        Xr = np.ascontiguousarray(big[:rows])
        Xd = torch.from_numpy(Xr).to(dev)
        outs = [torch.empty(rows, dtype=torch.float64, device=dev) for _ in probs]
        evb.evaluate_batch_problems(probs, Xd, evb.EvalScratch(), outs)
        torch.cuda.synchronize()
        got = evb.batched_evaluate_many(probs, Xr, sc)
        for g, w in zip(got, outs):
            assert np.array_equal(g, w.cpu().numpy()), rows
    # a non-contiguous view of a wider array
    wide = np.zeros((1024, 1003))
    wide[:, :1000] = X
    want = evb.batched_evaluate_many(probs, X, sc)
    for g, w in zip(evb.batched_evaluate_many(probs, wide[:, :1000], sc), want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("n_prob", [2, 3])
def test_problems_one_launch_bit_identical(config1, dev, n_prob):
    # several fp64 problems on one X in ONE launch (stages carry X once) == one launch per problem,
    # bit for bit (same tiles, K order, epilogue); with different shifts / rotations per problem
    o, m, X = config1
    o2, m2 = O.shift_rotation(8, 1000)
    specs = [(K.elliptic, o, m, 1.0), (K.rastrigin, o2, m2, 2.0), (K.ackley, o, m2, 3.0)][:n_prob]
    probs = [evb.ProblemInstance.base(k, oo, mm, b) for k, oo, mm, b in specs]
    want = [gpu_eval(p, X, dev) for p in probs]
    Xd = torch.from_numpy(X).to(dev)
    outs = [torch.empty(1024, dtype=torch.float64, device=dev) for _ in probs]
    n0 = evb.launch_count()
    evb.evaluate_batch_problems(probs, Xd, evb.EvalScratch(), outs)
    torch.cuda.synchronize()
    assert evb.launch_count() - n0 == 1
    for o_, w in zip(outs, want):
        assert np.array_equal(o_.cpu().numpy(), w)
    got = evb.batched_evaluate_many(probs, X)
    for g, w in zip(got, want):
        assert np.array_equal(g, w)


@pytest.mark.parametrize("n,dim", [(262144, 1000), (1024, 8192)])
def test_large_sizes_sampled(dev, n, dim):
    # maximum-size style batches (2.1 GB of X; a 537 MB rotation): checked on sampled rows against
    # the C restatement, and the fp64 result is deterministic across two launches
    rs = np.random.default_rng(dim)
    o = rs.uniform(-80, 80, dim)
    q, _ = np.linalg.qr(rs.standard_normal((dim, dim)))
    p = evb.ProblemInstance.base(K.rastrigin, o, q, 5.0)
    gen = torch.Generator(device=dev).manual_seed(dim)
    Xd = torch.rand((n, dim), dtype=torch.float64, device=dev, generator=gen) * 200.0 - 100.0
    out = torch.empty(n, dtype=torch.float64, device=dev)
    sc = evb.EvalScratch()
    evb.evaluate_batch(p, Xd, sc, out)
    out2 = torch.empty_like(out)
    evb.evaluate_batch(p, Xd, sc, out2)
    torch.cuda.synchronize()
    assert torch.equal(out, out2)
    rows = np.unique(np.concatenate([[0, n - 1], rs.integers(0, n, 14)]))
    Xs = Xd[torch.from_numpy(rows).to(dev)].cpu().numpy()
    ref = O.eval_batch(int(K.rastrigin), o, q, 5.0, Xs)
    assert rel_err(out.cpu().numpy()[rows], ref) <= 1e-10
    del Xd
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dim", [300, 1000])
def test_gemm_path_extreme_inputs(dev, dim):
    # the fused fp64 epilogue's fast cos(2 pi z) covers |z| < 2^16; larger and non-finite
    # arguments take the reference's own expression (warp-uniform switch): rows scaled far out of
    # the search domain, a NaN and an inf coordinate, against the C restatement — NaN / inf
    # positions identical, finite values within the path's 1e-10
    o, m = O.shift_rotation(7, dim)
    X = O.population(8, 70, dim)
    X[1] *= 1e3  # |z| beyond 2^16
    X[40:47] *= 3e2  # a whole 8-row epilogue group (and neighbours) around 2^16
    # far out (|z| ~ 1e7 .. 1e11): here the tensor-core summation order alone moves z by more than
    # cos(2 pi z) can absorb (~1e-15 |z|), so only NaN / inf agreement and finiteness are checked
    far = [2, 3]
    X[2] *= 1e5
    X[3] *= 1e9
    X[5, 7] = np.nan
    X[6, 11] = np.inf
    X[9, 0] = -np.inf
    kinds = [K.rastrigin, K.ackley, K.elliptic, K.griewank]
    for kind in kinds:
        p = evb.ProblemInstance.base(kind, o, m, 1.5)
        got = gpu_eval(p, X, dev)
        ref = O.eval_batch(int(kind), o, m, 1.5, X)
        assert np.array_equal(np.isnan(got), np.isnan(ref)), kind
        assert np.array_equal(np.isinf(got), np.isinf(ref)) and np.array_equal(got[np.isinf(ref)], ref[np.isinf(ref)])
        fin = np.isfinite(ref)
        fin[far] = False
        assert rel_err(got[fin], ref[fin]) <= 1e-10, kind
        assert np.all(np.isfinite(got[far]) == np.isfinite(ref[far])), kind
    # the multi-problem launch (its own 64 x 56 tiling) on the same population
    probs = [evb.ProblemInstance.base(k, o, m, 1.5) for k in kinds[:3]]
    Xd = torch.from_numpy(X).to(dev)
    outs = [torch.empty(X.shape[0], dtype=torch.float64, device=dev) for _ in probs]
    evb.evaluate_batch_problems(probs, Xd, evb.EvalScratch(), outs)
    torch.cuda.synchronize()
    for kind, o_ in zip(kinds[:3], outs):
        got = o_.cpu().numpy()
        ref = O.eval_batch(int(kind), o, m, 1.5, X)
        assert np.array_equal(np.isnan(got), np.isnan(ref)), kind
        fin = np.isfinite(ref)
        fin[far] = False
        assert rel_err(got[fin], ref[fin]) <= 1e-10, kind


@pytest.mark.parametrize("variant", [{"EVB_UMMA_ATMEM": "1"}, {"EVB_F32_MMA": "tf32"}])
@pytest.mark.parametrize("kind", [1, 5, 6])
def test_f32_tensor_core_variants(kind, variant):
    """The split-K fp32 kernel's selectable variants against the restatement at config 1's size
    (1e-4 relative): S_hi / S_lo as the MMA's A operand in TMEM (EVB_UMMA_ATMEM=1, tcgen05.mma with
    [a-tmem], 3xTF32), and the 3xTF32 shared-memory kernel (EVB_F32_MMA=tf32; the default is the
    fp16 split, 3xFP16).  The switches are read once per process, hence the subprocess."""
    import os
    import subprocess
    import sys
    import tempfile
    from pathlib import Path

    D, P = 1000, 1024
    o, m = O.shift_rotation(7, D)
    X = O.population(7, P, D)
    ref = O.eval_batch(kind, o, m, 0.0, X)
    code = f"""
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch, oracle as O, paper_2505_17430_b200 as evb
o, m = O.shift_rotation(7, {D}); X = O.population(7, {P}, {D})
p = evb.ProblemInstance.base({kind}, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32)
out = torch.empty({P}, dtype=torch.float32, device='cuda')
evb.evaluate_batch(p, torch.from_numpy(X.astype(np.float32)).cuda(), evb.EvalScratch(), out)
np.save(sys.argv[1], out.cpu().numpy())
"""
    with tempfile.TemporaryDirectory() as td:
        f = str(Path(td) / "v.npy")
        root = Path(__file__).resolve().parents[1]
        env = dict(os.environ, **variant)
        r = subprocess.run([sys.executable, "-c", code, f], cwd=str(root), capture_output=True, text=True, timeout=300,
                           env=env)
        assert r.returncode == 0, r.stderr[-2000:]
        got = np.load(f).astype(np.float64)
    err = np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref)))
    assert err <= 1e-4, err


def test_multi_problem_one_wave_variant_bit_identical():
    """The multi-problem K1 with 128-row blocks (EVB_K1M_BM=128: config 1 as one wave of 144 CTAs,
    32 x 56 warp tiles, ring refilled by warp 0; the switch is read once per process, hence the
    subprocesses) returns the same bits as the default 64-row kernel, device and host buffers,
    at config 1 and at a ragged size."""
    import os
    import subprocess
    import sys
    import tempfile
    from pathlib import Path

    code = """
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'oracle')
import numpy as np, torch, oracle as O, paper_2505_17430_b200 as evb
res = []
for (P, D) in ((1024, 1000), (333, 217)):
    o, m = O.shift_rotation(7, D); Xh = O.population(7, P, D)
    kinds = [evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
    probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in kinds]
    outs = [torch.empty(P, dtype=torch.float64, device='cuda') for _ in kinds]
    sc = evb.EvalScratch()
    evb.evaluate_batch_problems(probs, torch.from_numpy(Xh).cuda(), sc, outs)
    torch.cuda.synchronize()
    res.append(np.stack([t.cpu().numpy() for t in outs]).ravel())
    res.append(np.concatenate(evb.batched_evaluate_many(probs, Xh, sc)))
np.save(sys.argv[1], np.concatenate(res))
"""
    root = Path(__file__).resolve().parents[1]
    got = {}
    with tempfile.TemporaryDirectory() as td:
        for bm in ("64", "128"):
            f = str(Path(td) / f"v{bm}.npy")
            r = subprocess.run([sys.executable, "-c", code, f], cwd=str(root), capture_output=True, text=True,
                               timeout=300, env=dict(os.environ, EVB_K1M_BM=bm))
            assert r.returncode == 0, r.stderr[-2000:]
            got[bm] = np.load(f)
    assert np.array_equal(got["64"].view(np.uint64), got["128"].view(np.uint64))
    assert np.all(np.isfinite(got["128"]))


@pytest.mark.parametrize("dim", [300, 1000])
def test_f32_tensor_core_range_guard(dev, dim):
    """The 3xFP16 kernel's fp16 heads hold |x - o| < 65504.  Rows beyond that (or with a NaN / inf
    coordinate) are flagged by the split warps and recomputed in fp32 by the row block's last CTA:
    rows scaled 1e3 and 1e5 out of the search domain, a NaN and two inf coordinates, next to
    ordinary rows, against the fp64 restatement of the same float inputs (1e-4 relative, NaN / inf
    positions identical); a second launch on the same scratch (flags re-armed) with ordinary rows
    only; and a rotation whose scaled entries leave fp16's range (the problem stays on 3xTF32)."""
    o, m = O.shift_rotation(7, dim)
    X = O.population(8, 200, dim).astype(np.float32)
    X[1] *= 1e3
    X[130] *= 1e5
    X[5, 7] = np.nan
    X[6, 11] = np.inf
    X[199, 0] = -np.inf
    o32, m32 = o.astype(np.float32), m.astype(np.float32)
    sc = evb.EvalScratch()
    for kind in (K.elliptic, K.rastrigin, K.ackley, K.sphere):
        p = evb.ProblemInstance.base(kind, o32, m32, 1.5, dtype=evb.EVB_F32)
        for Xc in (X, O.population(9, 200, dim).astype(np.float32)):
            out = torch.empty(Xc.shape[0], dtype=torch.float32, device=dev)
            evb.evaluate_batch(p, torch.from_numpy(Xc).to(dev), sc, out)
            torch.cuda.synchronize()
            got = out.cpu().numpy().astype(np.float64)
            with np.errstate(all="ignore"):
                ref = O.eval_batch(int(kind), o32.astype(np.float64), m32.astype(np.float64), 1.5, Xc.astype(np.float64))
            assert np.array_equal(np.isnan(got), np.isnan(ref)), kind
            assert np.array_equal(np.isinf(got), np.isinf(ref)), kind
            fin = np.isfinite(ref)
            if kind == K.ackley and Xc is X:
                # far out the float spacing of z (~0.01 at 1e5) exceeds the period of cos(2 pi z):
                # the cosine sum of those rows is noise in any fp32 evaluation, only finiteness holds
                assert np.all(np.isfinite(got[[1, 130]]))
                fin[[1, 130]] = False
            assert rel_err(got[fin], ref[fin]) <= 1e-4, (kind, rel_err(got[fin], ref[fin]))
    # rotation entries of 1e3: 2^8 * 1e3 is not an fp16 number
    big = (m * 1e3).astype(np.float32)
    p = evb.ProblemInstance.base(K.elliptic, o32, big, 0.0, dtype=evb.EVB_F32)
    Xc = O.population(9, 200, dim).astype(np.float32)
    out = torch.empty(200, dtype=torch.float32, device=dev)
    for _ in range(2):
        evb.evaluate_batch(p, torch.from_numpy(Xc).to(dev), sc, out)
    torch.cuda.synchronize()
    ref = O.eval_batch(int(K.elliptic), o32.astype(np.float64), big.astype(np.float64), 0.0, Xc.astype(np.float64))
    assert rel_err(out.cpu().numpy().astype(np.float64), ref) <= 1e-4
