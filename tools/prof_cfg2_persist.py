"""Profiling driver: config 2 (SHADE, P=180, D=100, Ackley) generations in the persistent cluster
kernel (evb_de_generations), for ncu.  usage: python tools/prof_cfg2_persist.py [G]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_shade  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 50
P, D = 180, 100
o, m = O.shift_rotation(11, D)
prob = evb.ProblemInstance.base(evb.BaseKind.ackley, o, m, 0.0)
eng = DEEngine(preset_shade(0.11, P, 1.0), P, D)
rng = Rng.philox(11)
pop = torch.empty((P, D), dtype=torch.float64, device="cuda")
eng.init_population(pop, -100.0, 100.0, rng)
fit = torch.empty(P, dtype=torch.float64, device="cuda")
evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
torch.cuda.synchronize()
print("done", float(fit.min()))
