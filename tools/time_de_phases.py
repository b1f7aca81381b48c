"""Per-phase device times of one DE generation (CUDA events between the engine's kernels) over a
population-size sweep (tuning aid).  usage: python tools/time_de_phases.py D P1 P2 ..."""
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de, preset_shade  # noqa: E402

D = int(sys.argv[1])
dev = torch.device("cuda:0")
o, m = O.shift_rotation(13, D)
prob = evb.ProblemInstance.base(evb.BaseKind.sphere, o, m, 0.0)
for P in [int(a) for a in sys.argv[2:]]:
    for name, cfg in (("de", preset_de()), ("shade", preset_shade(0.11, 100, 1.0))):
        eng = DEEngine(cfg, P, D)
        rng = Rng.philox(5)
        pop = torch.empty((P, D), dtype=torch.float64, device=dev)
        eng.init_population(pop, -100.0, 100.0, rng)
        fit = torch.empty(P, dtype=torch.float64, device=dev)
        evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
        for _ in range(3):
            eng.generation(prob, pop, fit, -100.0, 100.0, rng)
        eng.phase_timing(True)
        ph = []
        for _ in range(7):
            eng.generation(prob, pop, fit, -100.0, 100.0, rng)
            ph.append(eng.phase_ms())
        eng.phase_timing(False)
        med = {k: round(statistics.median(p[k] for p in ph) * 1e3, 2) for k in ph[0]}
        print(f"P={P} D={D} {name}: {med}", flush=True)
