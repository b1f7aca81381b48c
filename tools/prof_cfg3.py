"""Config 3 (synchronous PSO gbest, fp64, D=1000, P=1024): a few iterations for an ncu launch list."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "oracle"))
import torch
import oracle as O
import paper_2505_17430_b200 as evb
from paper_2505_17430_b200.de import Rng
from paper_2505_17430_b200.pso import PSOEngine, config3
P, D = 1024, 1000
o, m = O.shift_rotation(13, D)
prob = evb.ProblemInstance.base(evb.BaseKind.elliptic, o, m, 0.0)
eng = PSOEngine(config3("gbest"), P, D, evb.EVB_F64)
rng = Rng.philox(13)
X = torch.empty((P, D), dtype=torch.float64, device="cuda")
V = torch.empty((P, D), dtype=torch.float64, device="cuda")
fit = torch.empty(P, dtype=torch.float64, device="cuda")
eng.init_uniform(X, -100.0, 100.0, rng)
eng.init_uniform(V, -20.0, 20.0, rng)
evb.evaluate_batch(prob, X, evb.EvalScratch(), fit)
eng.prepare(X, fit)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    eng.generation(prob, X, V, fit, -100.0, 100.0, rng)
torch.cuda.synchronize()
print("done")
