"""K8 on config 0's problem (D=10, P=100, scaled Rastrigin, `de` preset): device time per
generation of one run over 2000 generations (EVB_RUNS_SPLIT / EVB_RUNS_PROFILE apply; tuning aid)."""
import sys
sys.path.insert(0, "."); sys.path.insert(0, "oracle")
import torch
import oracle as O
import paper_2505_17430_b200 as evb
from paper_2505_17430_b200.de import preset_de
from paper_2505_17430_b200.runs import de_runs, run_keys
P, D, G = 100, 10, 2000
o, m = O.shift_rotation(42, D)
prob = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m * 0.0512, 0.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1
pops = torch.empty((n, P, D), dtype=torch.float64, device="cuda")
fits = torch.empty((n, P), dtype=torch.float64, device="cuda")
keys = run_keys(42, n)
de_runs(preset_de(), [prob] * n, keys, pops, fits, 20, -100.0, 100.0)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
de_runs(preset_de(), [prob] * n, keys, pops, fits, G, -100.0, 100.0)
b.record(); b.synchronize()
print(f"runs {n}: {a.elapsed_time(b) * 1e3 / G:.2f} us per generation; best {float(fits.min()):.4f}")
