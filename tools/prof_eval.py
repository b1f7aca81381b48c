"""Profiling driver: a few config-1 evaluate_batch launches (fp64 or fp32) for ncu."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402  (input generator only)
import paper_2505_17430_b200 as evb  # noqa: E402

dtype = sys.argv[1] if len(sys.argv) > 1 else "f64"
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 5
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 4
o, m = O.shift_rotation(7, 1000)
X = O.population(7, 1024, 1000)
if dtype == "f32":
    o, m, X = o.astype("float32"), m.astype("float32"), X.astype("float32")
p = evb.ProblemInstance.base(kind, o, m, 0.0, dtype=evb.EVB_F64 if dtype == "f64" else evb.EVB_F32)
sc = evb.EvalScratch()
Xd = torch.from_numpy(X).cuda()
out = torch.empty(1024, dtype=Xd.dtype, device="cuda")
for _ in range(reps):
    evb.evaluate_batch(p, Xd, sc, out)
torch.cuda.synchronize()
print("done", float(out[0]))
