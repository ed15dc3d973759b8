import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2406_10938_b200 as gpu
g = np.random.Generator(np.random.PCG64(77))
def sp(g, n, d):
    return np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)
data = sp(g, 60000, 128)
idx = gpu.build_index(data, gpu.LshParams(beta=0.2, k=20), seed=5)
Q = np.concatenate([np.full((24, 128), 255.0, np.float32) - g.integers(0, 3, (24, 128)).astype(np.float32), sp(g, 40, 128)])
for k in (1100, 1024, 1025, 600):
    os.environ["DETLSH_SLOW_DEFER_MIN"] = str(2**62)
    w = gpu.ck_ann_batch(idx, Q, k)
    os.environ["DETLSH_SLOW_DEFER_MIN"] = "0"
    o = gpu.ck_ann_batch(idx, Q, k)
    bad = np.where((o.ids != w.ids).any(1))[0]
    print(k, "bad queries", bad[:10], len(bad), "hits eq", np.array_equal(o.n_hits, w.n_hits), "dists eq", np.array_equal(o.dists, w.dists))
    for qq in bad[:2]:
        cols = np.where(o.ids[qq] != w.ids[qq])[0]
        print("  q", qq, "hits", w.n_hits[qq], "cols", cols[:8], len(cols), w.ids[qq][cols[:4]], o.ids[qq][cols[:4]], w.dists[qq][cols[:4]], o.dists[qq][cols[:4]])
k = 600
os.environ["DETLSH_SLOW_DEFER_MIN"] = "0"
o = gpu.ck_ann_batch(idx, Q, k)
os.environ["DETLSH_SLOW_DEFER_MIN"] = str(2**62)
w = gpu.ck_ann_batch(idx, Q, k)
for name, r in (("defer", o), ("inkernel", w)):
    true = np.sqrt(((Q[:, None, :].astype(np.float64) - data[r.ids[:, :5]].astype(np.float64)) ** 2).sum(-1))
    print(name, "max |dist - true| top5:", np.abs(true - r.dists[:, :5]).max(), "radius eq", np.array_equal(o.radius_used, w.radius_used), "cands eq", np.array_equal(o.candidates_seen, w.candidates_seen))
print(o.radius_used[:5], w.radius_used[:5], o.candidates_seen[:5], w.candidates_seen[:5])
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from oracle.bindings import Oracle, make_params
port = Oracle("port")
oi = port.build_index(data, make_params(beta=0.2, k=20), 5)
for name, r in (("defer", o), ("inkernel", w)):
    bad = []
    for qi in range(24):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], k)
        if not np.array_equal(r.ids[qi, :len(ids)], ids):
            bad.append(qi)
    print(name, "queries differing from the oracle:", bad)
