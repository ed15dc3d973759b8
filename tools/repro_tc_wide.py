"""Repro for the wide-row (R > 256) tensor-core verification path."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
d = int(sys.argv[1]) if len(sys.argv) > 1 else 784
n = int(sys.argv[2]) if len(sys.argv) > 2 else 120000
nq = int(sys.argv[3]) if len(sys.argv) > 3 else 300
g = np.random.Generator(np.random.PCG64(d))
x = np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)
Q = np.where(g.random((nq, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (nq, d)), 255)).astype(np.float32)
idx = D.build_index(x, D.LshParams(beta=0.1, k=50), seed=11)
print("built R", idx.row_u8(), flush=True)
ra = D.ck_ann_batch(idx, Q, 50)
rb = D.ck_ann_batch(idx, Q, 50, tensor_cores=False)
print("ids equal", np.array_equal(ra.ids, rb.ids), "dists equal", np.array_equal(ra.dists, rb.dists))
