"""Small build + queries (fast and general path) for compute-sanitizer runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, Q = gen.make("c2", n=20000, nq=6)
idx = D.build_index(base, D.LshParams(beta=0.1, k=20), seed=2)
r = D.ck_ann_batch(idx, Q, 20)
g = np.random.Generator(np.random.PCG64(1))
X = g.normal(0, 1, (3000, 16)).astype(np.float32)
idx2 = D.build_index(X, D.LshParams(K=8, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.01, k=5), seed=3)
r2 = D.ck_ann_batch(idx2, g.normal(0, 1, (6, 16)).astype(np.float32), 5)
print("ok", r.ids[0, :3], r2.radius_used)
