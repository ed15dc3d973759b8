"""Host-input (pinned) builds as bench.py's e2e leg runs them, with stage timings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, _ = gen.make("c2", nq=16)
pinned = torch.from_numpy(base).pin_memory().numpy()
p = D.LshParams(beta=0.1, k=50)
out = None
for i in range(6):
    t0 = time.perf_counter()
    out = D.build_index(pinned, p, seed=2, keep_codes=False)
    t1 = time.perf_counter()
    print(f"{(t1 - t0) * 1e3:.1f} ms", {k: round(v, 2) for k, v in out.build_timings().items()})
