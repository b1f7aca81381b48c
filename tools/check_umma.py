"""Quick fp32 tcgen05 (3xTF32) check against the C oracle: fused kinds, z-store kinds, ragged sizes."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

worst = 0.0
for D, P in ((1000, 1024), (200, 37), (257, 129)):
    o, m = O.shift_rotation(7, D)
    X = O.population(7, P, D)
    o32, m32, X32 = o.astype(np.float32), m.astype(np.float32), X.astype(np.float32)
    for kind in (1, 5, 6, 4, 3, 2, 7):
        p = evb.ProblemInstance.base(kind, o32, m32, 0.0, dtype=evb.EVB_F32)
        sc = evb.EvalScratch()
        Xd = torch.from_numpy(X32).cuda()
        out = torch.empty(P, dtype=torch.float32, device="cuda")
        evb.evaluate_batch(p, Xd, sc, out)
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.float64)
        ref = O.eval_batch(kind, o32, m32, 0.0, X32).astype(np.float64)
        err = float(np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))))
        worst = max(worst, err)
        print(f"D={D} P={P} kind={kind} max rel err {err:.3e}", flush=True)
print("WORST", worst)
