"""Build the C2 index once, run one batch of nq queries (for ncu captures)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
mode = sys.argv[3] if len(sys.argv) > 3 else "reference"
base, Q = gen.make(cfg, nq=nq)
idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=2, sample=mode)
t0 = time.time(); r = D.ck_ann_batch(idx, Q, 50); t1 = time.time()
print(f"{nq} queries {t1-t0:.4f}s {nq/(t1-t0):.1f} q/s; sum cands {int(r.candidates_seen.sum())}")
