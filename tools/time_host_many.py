"""Per-call latency of evb_evaluate_batch_host_many (config 1, fp64, three problems on one host
population); EVB_H2D_TRACE=1 prints the copy/kernel timeline of each call (tuning aid)."""
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, "oracle"); sys.path.insert(0, ".")
import oracle as O
import paper_2505_17430_b200 as evb
from paper_2505_17430_b200 import _lib
o, m = O.shift_rotation(7, 1000)
X = O.population(7, 1024, 1000)
Xh = torch.from_numpy(X).pin_memory()
kinds = [evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in kinds]
outh = [torch.empty(1024, dtype=torch.float64).pin_memory() for _ in kinds]
sc = evb.EvalScratch()
L = _lib.lib()
handles = (ctypes.c_void_p * 3)(*[p.handle.value for p in probs])
optrs = (ctypes.c_void_p * 3)(*[t.data_ptr() for t in outh])
def call():
    _lib.check(L.evb_evaluate_batch_host_many(handles, 3, sc.handle, ctypes.c_void_p(Xh.data_ptr()), 1024, 1000,
                                              optrs), "host_many")
n = int(sys.argv[1]) if len(sys.argv) > 1 else 400
for _ in range(20): call()
ts = []
for _ in range(n):
    t = time.perf_counter(); call(); ts.append(time.perf_counter() - t)
ts = np.array(ts) * 1e6
ref = [O.eval_batch(int(k), o, m, 0.0, X[:64]) for k in kinds]
err = max(float(np.max(np.abs(outh[i].numpy()[:64] - ref[i]) / np.maximum(1, np.abs(ref[i])))) for i in range(3))
print(f"host_many call us: p10 {np.percentile(ts,10):.1f} med {np.median(ts):.1f} p90 {np.percentile(ts,90):.1f} "
      f"-> {3 * 1024 / np.median(ts) * 1e6 / 1e6:.2f} M evals/s; max rel err (64 rows) {err:.2e}")
