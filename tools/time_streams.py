"""Config-1 step (elliptic + Rastrigin + Ackley on one X): three launches on one stream vs on
three streams (fork/join), L2 flushed between steps."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2505_17430_b200 as evb  # noqa: E402

o, m = O.shift_rotation(7, 1000)
X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
probs = [evb.ProblemInstance.base(k, o, m, 0.0) for k in (evb.BaseKind.elliptic, evb.BaseKind.rastrigin,
                                                          evb.BaseKind.ackley)]
scs = [evb.EvalScratch() for _ in probs]
outs = [torch.empty(1024, dtype=torch.float64, device="cuda") for _ in probs]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
main = torch.cuda.current_stream()
side = [torch.cuda.Stream() for _ in probs]


def step(concurrent):
    if not concurrent:
        for p, sc, out in zip(probs, scs, outs):
            evb.evaluate_batch(p, X, sc, out, main)
        return
    fork = torch.cuda.Event()
    fork.record(main)
    for p, sc, out, s in zip(probs, scs, outs, side):
        s.wait_event(fork)
        evb.evaluate_batch(p, X, sc, out, s)
        done = torch.cuda.Event()
        done.record(s)
        main.wait_event(done)


for concurrent in (False, True):
    ts = []
    for it in range(60):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        step(concurrent)
        b.record(main)
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    t = np.median(ts[10:])
    print(f"concurrent={concurrent}: step {t:.1f} us -> {3 * 1024 / (t * 1e-6) / 1e6:.2f} M evals/s")

outs3 = [torch.empty(1024, dtype=torch.float64, device="cuda") for _ in probs]
sc3 = evb.EvalScratch()
ts = []
for it in range(60):
    flush.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    evb.evaluate_batch_problems(probs, X, sc3, outs3, main)
    b.record(main)
    b.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
t = np.median(ts[10:])
print(f"one launch (evaluate_batch_problems): step {t:.1f} us -> {3 * 1024 / (t * 1e-6) / 1e6:.2f} M evals/s")
