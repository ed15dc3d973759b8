"""Back-to-back builds (as bench.py times them) to catch pool / stream regressions.
Prints per build: wall ms, the library's own 'total', and the time to drop the
previous index."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, _ = gen.make("c2", nq=16)
dev = torch.from_numpy(base).cuda()
p = D.LshParams(beta=0.1, k=50)
keep = "--keep" in sys.argv  # bench.py's pattern: the previous index lives until the next is built
modes = [m for m in sys.argv[1:] if not m.startswith("--")] or ["gpu", "gpu", "reference", "gpu"]
out = None
spikes = []
for mode in modes:
    rows = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if not keep:
            out = None  # drop the previous index
        t1 = time.perf_counter()
        out = D.build_index(dev, p, seed=2, sample=mode, borrow=True, keep_codes=False)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rows.append(f"{(t2 - t1) * 1e3:.1f}/{out.build_timings().get('total'):.1f}/drop {(t1 - t0) * 1e3:.1f}")
        if mode == "gpu" and (t2 - t1) > 0.009 or mode == "reference" and (t2 - t1) > 0.04:
            spikes.append((mode, {k: round(v, 2) for k, v in out.build_timings().items()}))
    print(mode, " | ".join(rows))
for sp in spikes:
    print("spike", sp)
