"""Back-to-back builds (as bench.py times them) to catch pool / stream regressions."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, _ = gen.make("c2", nq=16)
dev = torch.from_numpy(base).cuda()
p = D.LshParams(beta=0.1, k=50)
keep = D.build_index(dev, p, seed=2, sample=sys.argv[1] if len(sys.argv) > 1 else "reference", borrow=True, keep_codes=False)
for mode in ("gpu", "gpu", "reference", "gpu"):
    out = None
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        out = D.build_index(dev, p, seed=2, sample=mode, borrow=True, keep_codes=False)
    torch.cuda.synchronize()
    print(mode, f"{(time.perf_counter() - t0) / 5 * 1e3:.2f} ms per build", out.build_timings().get("total"))
