"""Profiling driver: one K8 launch (config 4 shape, `gens` generations) for ncu."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import preset_de  # noqa: E402
from paper_2505_17430_b200.runs import de_runs, run_keys  # noqa: E402

gens = int(sys.argv[1]) if len(sys.argv) > 1 else 50
n_runs, P, D = 64, 100, 50
probs = []
for r in range(n_runs):
    s, m = O.composition_components(4000 + r, D)
    probs.append(evb.ProblemInstance.composition(O.CONFIG4_KINDS, s, m, O.CONFIG4_SIGMA, O.CONFIG4_LAMBDA,
                                                 O.CONFIG4_BIAS, 0.0))
pops = torch.empty((n_runs, P, D), dtype=torch.float64, device="cuda")
fits = torch.empty((n_runs, P), dtype=torch.float64, device="cuda")
de_runs(preset_de(), probs, run_keys(64, n_runs), pops, fits, gens, -100.0, 100.0)
de_runs(preset_de(), probs, run_keys(64, n_runs), pops, fits, gens, -100.0, 100.0)
torch.cuda.synchronize()
print("done", float(fits.min()))
