"""Time the GPU exact kNN ground truth on a config (with and without the ANN bound)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
base, Q = gen.make(cfg, nq=nq)
k = 50
t0 = time.perf_counter(); ids, ds = D.brute_force_knn(base, Q, k); t1 = time.perf_counter()
print(f"{cfg}: brute force (sample threshold) {t1 - t0:.3f} s for {nq} queries")
idx = D.build_index(base, D.LshParams(beta=0.1, k=k), seed=2, sample="gpu")
res = D.ck_ann_batch(idx, Q, k)
bound = np.where(res.n_hits == k, res.dists[:, k - 1] ** 2 * (1 + 1e-12), np.inf)
t0 = time.perf_counter(); ids2, ds2 = D.brute_force_knn(base, Q, k, dist2_bound=bound); t1 = time.perf_counter()
print(f"{cfg}: brute force (ANN bound) {t1 - t0:.3f} s; identical: {np.array_equal(ids, ids2) and np.array_equal(ds, ds2)}")
