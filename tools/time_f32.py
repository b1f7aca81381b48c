"""fp32 config-1 batch (D=1000, P=1024) on the tensor-core kernel: relative fitness error against
the fp64 restatement for several kinds, and the device time per launch (back to back, CUDA events)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

D, P = 1000, 1024
o, m = O.shift_rotation(7, D)
X = O.population(7, P, D)
Xd = torch.from_numpy(X.astype(np.float32)).cuda()
sc = evb.EvalScratch()
out = torch.empty(P, dtype=torch.float32, device="cuda")
for kind in (evb.BaseKind.sphere, evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley,
             evb.BaseKind.griewank, evb.BaseKind.bent_cigar):
    p = evb.ProblemInstance.base(kind, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32)
    evb.evaluate_batch(p, Xd, sc, out)
    torch.cuda.synchronize()
    ref = O.eval_batch(int(kind), o, m, 0.0, X)
    got = out.cpu().numpy().astype(np.float64)
    err = np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref)))
    n = 300
    for _ in range(20):
        evb.evaluate_batch(p, Xd, sc, out)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        evb.evaluate_batch(p, Xd, sc, out)
    b.record()
    b.synchronize()
    print(f"{kind.name:12s} rel err {err:.2e}   {a.elapsed_time(b) * 1e3 / n:.2f} us per launch", flush=True)
