"""Config 0 (DE rand/1/bin, D=10, P=100): a few generations for an ncu launch list."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de  # noqa: E402

P, D = 100, 10
o, m = O.shift_rotation(42, D)
prob = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m * 0.0512, 0.0)
eng = DEEngine(preset_de(), P, D)
rng = Rng.philox(11)
pop = torch.empty((P, D), dtype=torch.float64, device="cuda")
fit = torch.empty(P, dtype=torch.float64, device="cuda")
eng.init_population(pop, -100.0, 100.0, rng)
evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    eng.generation(prob, pop, fit, -100.0, 100.0, rng)
torch.cuda.synchronize()
print("done")
