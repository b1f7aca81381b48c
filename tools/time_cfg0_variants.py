"""Config 0 (DE rand/1/bin, D=10, pop 100): graph-replayed generation time under env toggles of
the engine's kernel variants (tuning aid).  usage: python tools/time_cfg0_variants.py"""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402
from paper_2505_17430_b200.de import DEEngine, Rng, preset_de, preset_shade  # noqa: E402

dev = torch.device("cuda:0")


def run(cfg, P, D, kind, n=2000):
    o, m = O.shift_rotation(42, D)
    prob = evb.ProblemInstance.base(kind, o, m, 0.0)
    eng = DEEngine(cfg, P, D)
    rng = Rng.philox(42)
    pop = torch.empty((P, D), dtype=torch.float64, device=dev)
    eng.init_population(pop, -100.0, 100.0, rng)
    fit = torch.empty(P, dtype=torch.float64, device=dev)
    evb.evaluate_batch(prob, pop, evb.EvalScratch(), fit)
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, 20)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.generations(prob, pop, fit, -100.0, 100.0, rng, n)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3


VARS = [{}, {"EVB_DE_TRIAL_SCALAR": "1"}, {"EVB_DE_ORDER_RANK": "1"}, {"EVB_DE_SELECT_MULTI": "1"}]
for name, cfg, P, D, kind in (("config0", preset_de(), 100, 10, evb.BaseKind.rastrigin),
                              ("config2", preset_shade(0.11, 180, 1.0), 180, 100, evb.BaseKind.ackley)):
    for v in VARS:
        for k in ("EVB_DE_TRIAL_SCALAR", "EVB_DE_ORDER_RANK", "EVB_DE_SELECT_MULTI"):
            os.environ.pop(k, None)
        os.environ.update(v)
        print(f"{name} {v}: {run(cfg, P, D, kind):.2f} us/generation", flush=True)
