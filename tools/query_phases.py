"""Per-phase breakdown of the fast query kernel on a config (profiling hooks)."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
base, Q = gen.make(cfg, nq=nq)
idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=2)
lib = D.load()
D.ck_ann_batch(idx, Q, 50)
t0 = time.perf_counter()
D.ck_ann_batch(idx, Q, 50)
t1 = time.perf_counter()
lib.detlsh_profile_enable(1)
D.ck_ann_batch(idx, Q, 50)
lib.detlsh_profile_enable(0)
ph = np.zeros(8)
lib.detlsh_query_phase_cycles(C.c_void_p(ph.ctypes.data))
names = ["setup", "leaf_scan", "cut", "emission/flags (tc: bitmap)", "verify_topk (tc: tau rows + tau^2)", "output"]
tot = ph[:6].sum()
print(f"{cfg} nq={nq}: {nq/(t1-t0):.0f} q/s (unprofiled wall {1e3*(t1-t0):.1f} ms); "
      f"leaves={idx.tree(0).is_leaf.sum()} exact-round fallbacks={ph[6]:.0f} "
      f"exactly scored leaves/query={ph[7]/nq:.0f}")
for n_, v in zip(names, ph[:6]):
    print(f"  {n_:12s} {100*v/tot:5.1f}%  {v/nq/1e3:8.1f} kcycles/query (CTA thread-0 view)")
