"""Device time of the multi-problem K1 launch (config 1: three problems on one population), L2 flushed."""
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'oracle')
import numpy as np, torch, oracle as O, paper_2505_17430_b200 as evb
o, m = O.shift_rotation(7, 1000); X = torch.from_numpy(O.population(7, 1024, 1000)).cuda()
kinds=[evb.BaseKind.elliptic, evb.BaseKind.rastrigin, evb.BaseKind.ackley]
probs=[evb.ProblemInstance.base(k,o,m,0.0) for k in kinds]; outs=[torch.empty(1024,dtype=torch.float64,device='cuda') for _ in kinds]
flush=torch.empty(64<<20,dtype=torch.float32,device='cuda'); sc=evb.EvalScratch(); ts=[]
for it in range(40):
    flush.fill_(it); a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True); a.record()
    evb.evaluate_batch_problems(probs, X, sc, outs); b.record(); b.synchronize(); ts.append(a.elapsed_time(b)*1e3)
print("multi-problem K1 (3 problems):", np.mean(sorted(ts[5:])[5:-5]), "us")
