"""Fraction of tree-0 leaves the fast path's pass 1 finds not certainly
outside the radius (DETLSH_DEBUG_QUERY + profiling), for a config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
base, Q = gen.make(cfg, nq=nq)
idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=2)
lib = D.load()
D.ck_ann_batch(idx, Q, 50)
os.environ["DETLSH_DEBUG_QUERY"] = "1"
lib.detlsh_profile_enable(1)
D.ck_ann_batch(idx, Q, 50)
lib.detlsh_profile_enable(0)
