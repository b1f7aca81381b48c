import sys, time, ctypes
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import numpy as np, torch
import oracle as O
import paper_2505_17430_b200 as evb
from paper_2505_17430_b200 import _lib
o, m = O.shift_rotation(7, 1000)
X = O.population(7, 1024, 1000)
kinds = [evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in kinds]
sc = evb.EvalScratch()
Xh = torch.from_numpy(X).pin_memory()
outh = [torch.empty(1024, dtype=torch.float64).pin_memory() for _ in kinds]
L = _lib.lib()
handles = (ctypes.c_void_p * 3)(*[p.handle.value for p in probs])
optrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in outh])
def call():
    _lib.check(L.evb_evaluate_batch_host_many(handles, 3, sc.handle, ctypes.c_void_p(Xh.data_ptr()), 1024, 1000, optrs), "e2e")
def blocks(tag):
    for _ in range(5): call()
    torch.cuda.synchronize()
    r = []
    for b in range(5):
        t = time.perf_counter()
        for _ in range(40): call()
        torch.cuda.synchronize()
        r.append((time.perf_counter() - t) / 40 * 1e6)
    print(tag, [round(x, 1) for x in r], flush=True)
blocks("fresh scratch")
Xd = torch.from_numpy(X).cuda(); out = torch.empty(1024, dtype=torch.float64, device="cuda")
for _ in range(50):
    evb.evaluate_batch(probs[0], Xd, sc, out)
torch.cuda.synchronize()
blocks("after device evaluate_batch on the same scratch")
sc2 = evb.EvalScratch()
blocks("same scratch again")
