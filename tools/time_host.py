"""Per-call latency of evb_evaluate_batch_host (config 1, fp64) vs a plain pinned H2D copy of X."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import oracle as O
import paper_2505_17430_b200 as evb
from paper_2505_17430_b200 import _lib
o, m = O.shift_rotation(7, 1000)
X = O.population(7, 1024, 1000)
Xh = torch.from_numpy(X).pin_memory()
outh = torch.empty(1024, dtype=torch.float64).pin_memory()
p = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m, 0.0)
sc = evb.EvalScratch()
L = _lib.lib()
def call():
    _lib.check(L.evb_evaluate_batch_host(p.handle, sc.handle, ctypes.c_void_p(Xh.data_ptr()), 1024, 1000,
                                         ctypes.c_void_p(outh.data_ptr())), "host")
for _ in range(20): call()
ts = []
for _ in range(500):
    t = time.perf_counter(); call(); ts.append(time.perf_counter() - t)
ts = np.array(ts) * 1e6
Xd = torch.empty_like(Xh, device="cuda")
cs = []
for _ in range(200):
    torch.cuda.synchronize(); t = time.perf_counter(); Xd.copy_(Xh, non_blocking=True); torch.cuda.synchronize(); cs.append(time.perf_counter() - t)
cs = np.array(cs) * 1e6
Xdd = torch.from_numpy(X).cuda(); out = torch.empty(1024, dtype=torch.float64, device="cuda")
ks = []
for _ in range(200):
    torch.cuda.synchronize(); t = time.perf_counter(); evb.evaluate_batch(p, Xdd, sc, out); torch.cuda.synchronize(); ks.append(time.perf_counter() - t)
ks = np.array(ks) * 1e6
print(f"host call us: p10 {np.percentile(ts,10):.1f} med {np.median(ts):.1f} p90 {np.percentile(ts,90):.1f} | "
      f"pinned H2D 8.19MB us med {np.median(cs):.1f} ({8.192e6/np.median(cs)/1e3:.1f} GB/s) | device eval us med {np.median(ks):.1f}")
