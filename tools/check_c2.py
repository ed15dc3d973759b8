"""Full-size C2 parity spot check: GPU vs the C oracle on a few queries."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
from oracle.bindings import Oracle, make_params
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 20
base, Q = gen.make(cfg, nq=nq)
p = D.LshParams(beta=0.1, k=50)
t0 = time.time(); idx = D.build_index(base, p, seed=2); print("gpu build", time.time()-t0, flush=True)
t0 = time.time(); r = D.ck_ann_batch(idx, Q, 50); t1 = time.time(); print("gpu query", t1-t0, flush=True)
orc = Oracle("port")
t0 = time.time(); oi = orc.build_index(base, make_params(beta=0.1, k=50), 2); print("oracle build", time.time()-t0, flush=True)
print("rmin", idx.params.r_min, oi.params.r_min)
bad = 0
t0 = time.time()
for i in range(nq):
    ids, ds, rad, cs = oi.ck_ann(Q[i], 50)
    ok = np.array_equal(r.ids[i], ids) and np.array_equal(r.dists[i], ds) and rad == r.radius_used[i] and cs == r.candidates_seen[i]
    bad += not ok
    if not ok and bad < 3:
        print("MISMATCH", i, r.ids[i][:8], ids[:8], r.dists[i][:4], ds[:4], rad, r.radius_used[i], cs, r.candidates_seen[i])
print("oracle queries", time.time()-t0, "mismatches", bad, "of", nq)
