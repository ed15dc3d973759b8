"""Back-to-back reference-sample builds of one config as bench.py times them
(the previous index alive until the next is built), with the library's stage
timings per build.  Usage: python tools/build_repeat_cfg.py [config] [reps] [host]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
host = len(sys.argv) > 3 and sys.argv[3] == "host"
base, _ = gen.make(cfg, nq=16)
src = torch.from_numpy(base).pin_memory().numpy() if host else torch.from_numpy(base).cuda()
kw = {} if host else dict(borrow=True)
p = D.LshParams(beta=0.1, k=50)
out = None
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = D.build_index(src, p, seed=2, keep_codes=False, **kw)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    st = out.build_timings()
    print(f"{cfg} build {r}: {dt:.1f} ms", {k: round(v, 1) for k, v in st.items()}, flush=True)
