#!/bin/bash
# A/B of the multi-problem K1 row-block height (EVB_K1M_BM=64|128): device time, bit-equality, e2e
for bm in 64 128; do
  echo "== EVB_K1M_BM=$bm"; EVB_K1M_BM=$bm python tools/time_multi.py
done
python - <<'PY'
import os, subprocess, sys
sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
code = r'''
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np, torch, oracle as O, paper_2505_17430_b200 as evb
o, m = O.shift_rotation(7, 1000); X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
kinds=[evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
probs=[evb.ProblemInstance.base(k,o,m,0.0) for k in kinds]; outs=[torch.empty(1024,dtype=torch.float64,device='cuda') for _ in kinds]
sc=evb.EvalScratch(); evb.evaluate_batch_problems(probs, X, sc, outs); torch.cuda.synchronize()
np.save(sys.argv[1], np.stack([t.cpu().numpy() for t in outs]))
'''
for bm in ("64", "128"):
    subprocess.run([sys.executable, "-c", code, f"/tmp/k1m_{bm}.npy"], env=dict(os.environ, EVB_K1M_BM=bm), check=True)
import numpy as np
a, b = np.load("/tmp/k1m_64.npy"), np.load("/tmp/k1m_128.npy")
print("bit-identical 64 vs 128:", bool((a.view(np.uint64) == b.view(np.uint64)).all()), a[:, :2])
PY
