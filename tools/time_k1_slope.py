"""K1 fixed cost vs mainloop rate: elliptic evaluate_batch at shapes with the same 288 tiles of
64 x 56 but K = 1000 / 2000 / 4000 (P x D = 1024 x 1000, 512 x 2000, 256 x 4000), L2 flushed.
The slope gives the mainloop's DMMA rate, the intercept the per-launch fixed cost (fill,
epilogue, tail)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

kind = evb.BaseKind[sys.argv[1]] if len(sys.argv) > 1 else evb.BaseKind.elliptic
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch()
res = []
for P, D in ((1024, 1000), (512, 2000), (256, 4000)):
    rng = np.random.default_rng(1)
    o = rng.uniform(-80, 80, D)
    m = np.linalg.qr(rng.standard_normal((D, D)))[0]
    X = torch.from_numpy(rng.uniform(-100, 100, (P, D))).cuda()
    out = torch.empty(P, dtype=torch.float64, device="cuda")
    p = evb.ProblemInstance.base(kind, o, m, 0.0)
    ts = []
    for it in range(40):
        flush.fill_(it)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        evb.evaluate_batch(p, X, sc, out)
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    t = float(np.median(ts[10:]))
    res.append((D, t))
    print(f"{kind.name} P={P} D={D}: {t:.1f} us  {2.0 * P * D * D / t / 1e6:.2f} TF/s", flush=True)
(k0, t0), (k1, t1), (k2, t2) = res
slope = (t2 - t0) / (k2 - k0)
print(f"per-1000-K mainloop {slope * 1000:.1f} us -> {2.0 * 1024 * 1000 * 1000 / (slope * 1000) / 1e6:.2f} TF/s; "
      f"fixed {t0 - slope * k0:.1f} us")
