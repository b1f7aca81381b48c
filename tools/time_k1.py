"""Median device time of evaluate_batch (config 1, fp64) per objective kind, L2 flushed between
launches; run once per EVB_F64_KERNEL variant (the variant is read once per process)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

o, m = O.shift_rotation(7, 1000)
X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch()
out = torch.empty(1024, dtype=torch.float64, device="cuda")
res = {}
for kind in (evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley):
    p = evb.ProblemInstance.base(kind, o, m, 0.0)
    ts = []
    for it in range(60):
        flush.fill_(it)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        evb.evaluate_batch(p, X, sc, out)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res[kind.name] = np.median(ts[10:])
tf = [2.048e9 / (t * 1e-6) / 1e12 for t in res.values()]
print(" ".join(f"{k} {v:.1f}us" for k, v in res.items()), f"| mean {np.mean(list(res.values())):.1f}us",
      f"{np.mean(tf):.2f} TF/s")
