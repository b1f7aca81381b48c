"""fp32 config-1 evaluation: host cost per evaluate_batch call and device time per step (one
event pair around the step's three launches vs one pair per launch).  Tuning aid."""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

D, P = 1000, 1024
o, m = O.shift_rotation(7, D)
X = O.population(7, P, D).astype(np.float32)
kinds = (evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley)
probs = [evb.ProblemInstance.base(k, o.astype(np.float32), m.astype(np.float32), 0.0, dtype=evb.EVB_F32) for k in kinds]
sc = evb.EvalScratch()
Xd = torch.from_numpy(X).cuda()
outs = [torch.empty(P, dtype=torch.float32, device="cuda") for _ in kinds]
st = torch.cuda.current_stream()
for _ in range(20):
    for p, f in zip(probs, outs):
        evb.evaluate_batch(p, Xd, sc, f, st)
torch.cuda.synchronize()
n = 300
t0 = time.perf_counter()
for _ in range(n):
    for p, f in zip(probs, outs):
        evb.evaluate_batch(p, Xd, sc, f, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host enqueue per call {1e6 * (t1 - t0) / (3 * n):.1f} us; wall per call incl. drain {1e6 * (t2 - t0) / (3 * n):.1f} us")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(st)
for _ in range(n):
    for p, f in zip(probs, outs):
        evb.evaluate_batch(p, Xd, sc, f, st)
b.record(st)
torch.cuda.synchronize()
print(f"device per launch, back to back: {1e3 * a.elapsed_time(b) / (3 * n):.2f} us")
