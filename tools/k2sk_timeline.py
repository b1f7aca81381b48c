"""Per-CTA phase timeline of the split-K fp32 tcgen05 kernel (EVB_K1_TIMELINE=1 hook): entry,
first stage consumed by the MMA issuer, accumulator complete, partials written / z parked, exit.
Columns: c, start, first, accfull, partials written, end, last-column-block flag, exchange done.
Tuning aid."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
os.environ["EVB_K1_TIMELINE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

kind = evb.BaseKind[sys.argv[1]] if len(sys.argv) > 1 else evb.BaseKind.rastrigin
o, m = O.shift_rotation(7, 1000)
X = torch.from_numpy(O.population(7, 1024, 1000).astype(np.float32)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch()
out = torch.empty(1024, dtype=torch.float32, device="cuda")
p = evb.ProblemInstance.base(kind, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32)
f = ROOT / "gpurun_out" / "k2_ts.csv"
if f.exists():
    f.unlink()
for it in range(6):
    if os.environ.get("K2_NOFLUSH") is None:
        flush.fill_(it)
    torch.cuda.synchronize()
    evb.evaluate_batch(p, X, sc, out)
    torch.cuda.synchronize()
runs = f.read_text().strip().split("end\n")
for r in runs[2:]:
    a = np.array([[int(x) for x in ln.split(",")] for ln in r.strip().split("\n") if ln and ln != "end"], np.float64)
    t0 = a[:, 1].min()

    def q(v):
        return f"{np.min(v) / 1e3:.1f}/{np.median(v) / 1e3:.1f}/{np.max(v) / 1e3:.1f}" if len(v) else "-"

    ex = a[:, 7] > 0  # the K halves exchanged (split-K launches)
    xt = np.where(ex, a[:, 7], a[:, 3])
    print(f"{kind.name}: start {q(a[:, 1] - t0)} | first stage {q(a[:, 2] - a[:, 1])} | mainloop {q(a[:, 3] - a[:, 2])}"
          f" | exchange {q(xt - a[:, 3])} | terms+partials {q(a[:, 4] - xt)} | combine {q((a[:, 5] - a[:, 4])[a[:, 6] == 1])}"
          f" | end {np.max(a[:, 5] - t0) / 1e3:.1f} us")
