"""Quick timing probe (not the bench): C2 build stages + query throughput."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
t0 = time.time()
base, Q = gen.make(cfg, nq=nq)
print(f"gen {cfg} {base.shape} {time.time()-t0:.1f}s", flush=True)
p = D.LshParams(beta=0.1, k=50)
dev = torch.from_numpy(base).cuda()
for mode in ("reference", "gpu"):
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.time()
        idx = D.build_index(dev, p, seed=2, sample=mode, borrow=True)
        torch.cuda.synchronize(); t1 = time.time()
        print(f"build[{mode}] {1e3*(t1-t0):.1f} ms -> {base.shape[0]/(t1-t0)/1e6:.2f} Mpts/s", idx.build_timings(), flush=True)
print("r_min", idx.params.r_min, "leaves", [int(idx.tree(i).is_leaf.sum()) for i in range(1)])
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.time()
    r = D.ck_ann_batch(idx, Q, 50)
    torch.cuda.synchronize(); t1 = time.time()
    print(f"query {nq}: {t1-t0:.3f}s -> {nq/(t1-t0):.1f} q/s; slow-path frac {np.mean(r.radius_used != idx.params.r_min):.3f} cands {r.candidates_seen[:3]}", flush=True)
