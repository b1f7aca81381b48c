import sys, numpy as np, torch
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import oracle as O
import paper_2505_17430_b200 as evb
K = evb.BaseKind
o, m = O.shift_rotation(7, 1000)
X = O.population(7, 1024, 1000)
for kind in (K.elliptic, K.rastrigin, K.ackley, K.sphere):
    p = evb.ProblemInstance.base(kind, o, m, 10.0)
    sc = evb.EvalScratch()
    Xd = torch.from_numpy(X).cuda()
    out = torch.empty(1024, dtype=torch.float64, device="cuda")
    evb.evaluate_batch(p, Xd, sc, out)
    want = out.cpu().numpy()
    sc2 = evb.EvalScratch()
    for it in range(3):
        got = evb.batched_evaluate(p, X, sc2)
        d = np.abs(got - want) / np.abs(want)
        print(int(kind), it, "ndiff", int((got != want).sum()), "maxrel", d.max(), "first", np.nonzero(got != want)[0][:8])
