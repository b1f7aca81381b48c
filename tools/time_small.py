"""Device time of the small-D exact-order evaluation (config-2 and config-0 shapes), warm L2,
20 launches per CUDA graph, replays averaged (tuning aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, torch
import oracle as O
import paper_2505_17430_b200 as evb
sc = evb.EvalScratch()
for (P, D, kind) in ((180, 100, "ackley"), (100, 10, "rastrigin"), (100, 50, "rastrigin"), (1024, 100, "ackley"),
                     (180, 160, "ackley")):
    o, m = O.shift_rotation(11, D)
    X = torch.from_numpy(O.population(11, P, D)).cuda()
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    p = evb.ProblemInstance.base(getattr(evb.BaseKind, kind), o, m, 0.0)
    for _ in range(20):
        evb.evaluate_batch(p, X, sc, out)
    # device time: 20 launches captured in a CUDA graph, replayed (host launch cost excluded)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            evb.evaluate_batch(p, X, sc, out, s)
    g.replay(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    a.record()
    for _ in range(reps):
        g.replay()
    b.record(); b.synchronize()
    n = 20 * reps
    ref = O.eval_batch(int(getattr(evb.BaseKind, kind)), o, m, 0.0, X.cpu().numpy()[:16])
    err = float(np.max(np.abs(out.cpu().numpy()[:16] - ref) / np.maximum(1, np.abs(ref))))
    print(f"P={P} D={D} {kind}: {a.elapsed_time(b) * 1e3 / n:.2f} us per launch (graph), err {err:.1e}")
