"""Per-CTA phase timeline of K1 (EVB_K1_TIMELINE=1 hook): globaltimer stamps at entry, first
stage landed, mainloop end, epilogue terms end (ticket), exit.  Tuning aid."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
os.environ["EVB_K1_TIMELINE"] = "1"
import numpy as np, torch
import oracle as O
import paper_2505_17430_b200 as evb
kind = evb.BaseKind[sys.argv[1]] if len(sys.argv) > 1 else evb.BaseKind.rastrigin
o, m = O.shift_rotation(7, 1000)
X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch(); out = torch.empty(1024, dtype=torch.float64, device="cuda")
p = evb.ProblemInstance.base(kind, o, m, 0.0)
f = ROOT / "gpurun_out" / "k1_ts.csv"
if f.exists(): f.unlink()
for it in range(6):
    flush.fill_(it); torch.cuda.synchronize()
    evb.evaluate_batch(p, X, sc, out); torch.cuda.synchronize()
runs = f.read_text().strip().split("end\n")
for r in runs[2:]:
    a = np.array([[int(x) for x in l.split(",")] for l in r.strip().split("\n") if l and l != "end"], dtype=np.float64)
    t0 = a[:, 1].min()
    st, fl, ml, te, ex = a[:, 1] - t0, a[:, 2] - a[:, 1], a[:, 3] - a[:, 2], a[:, 4] - a[:, 3], a[:, 5] - a[:, 4]
    last = a[:, 6] == 1
    q = lambda v: f"{np.min(v)/1e3:.1f}/{np.median(v)/1e3:.1f}/{np.max(v)/1e3:.1f}"
    print(f"{kind.name}: start {q(st)} | fill {q(fl)} | mainloop {q(ml)} | terms {q(te)} | "
          f"combine(last) {q(ex[last])} other {q(ex[~last])} | end {np.max(a[:,5]-t0)/1e3:.1f} us "
          f"(mainloop-end max {np.max(a[:,3]-t0)/1e3:.1f})")
