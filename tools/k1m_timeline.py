"""Per-CTA phase timeline of the multi-problem K1 (three config-1 problems, EVB_K1_TIMELINE=1):
entry, first stage, mainloop end, group-0 exit; CTAs split into waves by start time.  Tuning aid."""
import os, sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
os.environ["EVB_K1_TIMELINE"] = "1"
import numpy as np, torch
import oracle as O
import paper_2505_17430_b200 as evb
o, m = O.shift_rotation(7, 1000)
X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
kinds = [evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in kinds]
outs = [torch.empty(1024, dtype=torch.float64, device="cuda") for _ in kinds]
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
sc = evb.EvalScratch()
f = ROOT / "gpurun_out" / "k1m_ts.csv"
if f.exists(): f.unlink()
for it in range(5):
    flush.fill_(it); torch.cuda.synchronize()
    evb.evaluate_batch_problems(probs, X, sc, outs); torch.cuda.synchronize()
for r in f.read_text().strip().split("end\n")[2:]:
    a = np.array([[int(x) for x in l.split(",")] for l in r.strip().split("\n") if l and l != "end"],
                 dtype=np.float64)
    if a.size == 0:
        continue
    t0 = a[:, 1].min()
    st = (a[:, 1] - t0) / 1e3
    w2 = st > 20.0
    q = lambda v: f"{np.min(v):.1f}/{np.median(v):.1f}/{np.max(v):.1f}"
    for name, sel in (("wave1", ~w2), ("wave2", w2)):
        b = a[sel]
        print(f"{name} ({sel.sum()} CTAs): start {q((b[:,1]-t0)/1e3)} | fill {q((b[:,2]-b[:,1])/1e3)} | "
              f"mainloop {q((b[:,3]-b[:,2])/1e3)} | epilogue {q((b[:,4]-b[:,3])/1e3)} | end {q((b[:,4]-t0)/1e3)}")
    print("kernel end", f"{(a[:,4].max()-t0)/1e3:.1f} us")
