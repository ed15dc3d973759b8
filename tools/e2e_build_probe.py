"""Stage timings of the end-to-end (pinned host input) build vs the
device-resident build of a config.  Usage: python tools/e2e_build_probe.py [config] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
base, _ = gen.make(cfg, nq=0)
pin = torch.from_numpy(base).pin_memory().numpy()
dev = torch.from_numpy(base).cuda()
p = D.LshParams(beta=0.1, k=50)
for name, src, kw in (("device", dev, dict(borrow=True)), ("host_pinned", pin, {})):
    for r in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ix = D.build_index(src, p, seed=2, keep_codes=False, **kw)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) * 1e3
        if r == reps - 1:
            st = ix.build_timings()
            print(name, f"{dt:.2f} ms", {k: round(v, 2) for k, v in st.items()})
        del ix
