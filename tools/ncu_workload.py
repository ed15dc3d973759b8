"""One build + one full query batch of a config, for ncu captures of the
product kernels (nothing is timed here).  Usage: python tools/ncu_workload.py [config] [nq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else None
base, Q = gen.make(cfg, nq=nq)
X = torch.from_numpy(base).cuda()
idx = D.build_index(X, D.LshParams(beta=0.1, k=50), seed=2, borrow=True, keep_codes=False)
Qd = torch.from_numpy(Q).cuda()
k = 50
ids = torch.empty((Q.shape[0], k), dtype=torch.int32, device="cuda")
ds = torch.empty((Q.shape[0], k), dtype=torch.float64, device="cuda")
D.ck_ann_device(idx, Qd, k, ids, ds)
torch.cuda.synchronize()
print("done", cfg, Q.shape[0])
