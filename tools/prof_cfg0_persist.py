"""Config 0 (DE rand/1/bin, D=10, P=100) generations in the persistent cluster kernel
(evb_de_generations): device time per generation; EVB_DE_PERSIST_PROFILE=1 prints CTA 0's cycles per
phase.  usage: python tools/prof_cfg0_persist.py [G]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
P, D = 100, 10
o, m = O.shift_rotation(42, D)
prob = evb.ProblemInstance.base(evb.BaseKind.rastrigin, o, m * 0.0512, 0.0)
eng = DEEngine(preset_de(), P, D)
rng = Rng.philox(42)
pop = torch.empty((P, D), dtype=torch.float64, device="cuda")
fit = torch.empty(P, dtype=torch.float64, device="cuda")
eng.init_population(pop, -100.0, 100.0, rng)
evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
eng.generations(prob, pop, fit, -100.0, 100.0, rng, G)
b.record()
b.synchronize()
print(f"config 0 persistent: {a.elapsed_time(b) * 1e3 / G:.2f} us per generation, best {float(fit.min()):.6g}")
