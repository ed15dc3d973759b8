import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from oracle.bindings import Oracle
n = int(sys.argv[1]); d = int(sys.argv[2])
g = np.random.Generator(np.random.PCG64(5))
x = np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)
fam = D.sample_hash_family(d, 16, 4, 3)
got = D.project_dataset(fam, x)
want = Oracle("port").project_dataset(fam, x[:2000])
print("stage ok", np.array_equal(got[:, :2000].view(np.uint32), want.view(np.uint32)))
idx = D.build_index(x, D.LshParams(beta=0.1, k=20), seed=11)
print("build ok", idx.params.r_min)
