"""Time the fp32 evaluation (config-1 shape, Rastrigin)."""
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
X = O.population(7, 1024, 1000)
p = evb.ProblemInstance.base(5, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32)
sc = evb.EvalScratch()
Xd = torch.from_numpy(X.astype(np.float32)).cuda()
out = torch.empty(1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    evb.evaluate_batch(p, Xd, sc, out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(50):
    evb.evaluate_batch(p, Xd, sc, out)
b.record()
torch.cuda.synchronize()
print("ms per evaluate_batch", a.elapsed_time(b) / 50)
