import os, sys
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2406_10938_b200 as gpu
from oracle.bindings import Oracle, make_params
g = np.random.Generator(np.random.PCG64(77))
def sp(g, n, d):
    return np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)
data = sp(g, 60000, 128)
idx = gpu.build_index(data, gpu.LshParams(beta=0.2, k=20), seed=5)
Q = np.concatenate([np.full((24, 128), 255.0, np.float32) - g.integers(0, 3, (24, 128)).astype(np.float32), sp(g, 40, 128)])
port = Oracle("port")
oi = port.build_index(data, make_params(beta=0.2, k=20), 5)
orcs = {}
def check(tag, k, r):
    if k not in orcs:
        orcs[k] = [oi.ck_ann(Q[qi], k) for qi in range(Q.shape[0])]
    orc = orcs[k]
    bad = [qi for qi in range(Q.shape[0]) if not np.array_equal(r.ids[qi, :len(orc[qi][0])], orc[qi][0])]
    print(tag, k, "differ from oracle:", bad, flush=True)
for k, mode in [(600, "in"), (1100, "in"), (600, "in"), (600, "in"), (1100, "def"), (600, "in"), (600, "in")]:
    os.environ["DETLSH_SLOW_DEFER_MIN"] = "0" if mode == "def" else str(2**62)
    check(mode, k, gpu.ck_ann_batch(idx, Q, k))
