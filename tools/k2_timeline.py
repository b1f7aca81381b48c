"""Per-CTA phase timeline of the fp32 tcgen05 kernel (EVB_K1_TIMELINE=1 hook): entry, first
stage landed (MMA issuer), accumulator complete (epilogue start), terms done, exit.  Tuning aid."""
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
X = torch.from_numpy(O.population(7, 1024, 1000).astype(np.float32)).cuda()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch(); out = torch.empty(1024, dtype=torch.float32, device="cuda")
p = evb.ProblemInstance.base(kind, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32)
f = ROOT / "gpurun_out" / "k2_ts.csv"
if f.exists(): f.unlink()
for it in range(6):
    flush.fill_(it); torch.cuda.synchronize()
    evb.evaluate_batch(p, X, sc, out); torch.cuda.synchronize()
runs = f.read_text().strip().split("end\n")
for r in runs[2:]:
    a = np.array([[int(x) for x in l.split(",")] for l in r.strip().split("\n") if l and l != "end"], dtype=np.float64)
    t0 = a[:, 1].min()
    q = lambda v: f"{np.min(v)/1e3:.1f}/{np.median(v)/1e3:.1f}/{np.max(v)/1e3:.1f}"
    last = a[:, 6] == 1
    print(f"{kind.name} fp32: start {q(a[:,1]-t0)} | first stage {q(a[:,2]-a[:,1])} | mainloop {q(a[:,3]-a[:,2])} | "
          f"terms {q(a[:,4]-a[:,3])} | combine(last) {q((a[:,5]-a[:,4])[last])} | end {np.max(a[:,5]-t0)/1e3:.1f} us")
