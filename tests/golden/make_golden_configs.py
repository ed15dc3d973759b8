"""Full-size golden fixtures for BASELINE.json's configs, generated from the REAL
reference (oracle/_ref/libdetlsh_ref.so = /root/reference/proj/src compiled by
`make -C oracle ref`).  Run in the dev container (takes ~15 min, ~25 GB RAM):

    python tests/golden/make_golden_configs.py [c1 c2 c3 c4]

Inputs are NOT stored: they are regenerated from the seeded generators in
paper_2406_10938_b200/data.py (numpy PCG64).  Each fixture records what the
reference's build_index (index.cpp:212-218) and ck_ann (index.cpp:292-331)
return on them: the derived params and r_min, the breakpoint table, a SHA-256
of every DE-Tree's node stream (same layout as tests/golden_util.tree_hash),
and ids / distances / radius_used / candidates_seen / hit counts for the first
`nq` held-out queries.  The GPU tests (tests/test_gpu_configs.py) rebuild the
index with the CUDA path and compare bit for bit.
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.bindings import Oracle, make_params  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

# config -> (seed of build_index, queries pinned); every config: K=16, L=4,
# N_r=256, sample 0.1, leaf 128, c=1.5, beta=0.1, k=50
CONFIGS = {
    "c1": (1, 1000),
    "c2": (2, 1000),
    "c3": (3, 200),
    "c4": (4, 200),
}
K_NN = 50
BETA = 0.1


def fixture_path(cfg):
    return os.path.join(HERE, f"cfg_{cfg}.npz")


def main(names):
    from golden_util import tree_hash
    ref = Oracle("reference")
    threads = os.cpu_count() or 1
    for cfg in names:
        seed, nq = CONFIGS[cfg]
        t0 = time.time()
        base, Q = gen.make(cfg)
        Q = np.ascontiguousarray(Q[:nq])
        t1 = time.time()
        p = make_params(beta=BETA, k=K_NN)
        idx = ref.build_index(base, p, seed)
        t2 = time.time()
        ids, ds, nh, rad, cs, secs = idx.ck_ann_batch(Q, K_NN, threads=threads)
        p = idx.params
        trees = [idx.tree_export(i) for i in range(p.L)]
        out = dict(
            config=cfg, n=base.shape[0], d=base.shape[1], nq=nq, seed=seed,
            params=np.array([p.K, p.L, p.c, p.beta, p.epsilon, p.alpha1, p.alpha2, p.n_regions,
                             p.sample_fraction, p.leaf_capacity, p.r_min, p.k], np.float64),
            table=idx.table(), ids=ids, dists=ds, radius=rad, cands=cs, n_hits=nh,
            tree_nodes=np.array([len(t.is_leaf) for t in trees]),
            tree_hash=np.array([tree_hash(t) for t in trees]),
            ref_build_s=t2 - t1, ref_query_s=secs, ref_threads=threads,
        )
        np.savez_compressed(fixture_path(cfg), **out)
        print(f"{cfg}: gen {t1 - t0:.1f}s build {t2 - t1:.1f}s queries {secs:.1f}s "
              f"r_min {p.r_min} nodes {out['tree_nodes'].tolist()}", flush=True)
        del idx, base


if __name__ == "__main__":
    main(sys.argv[1:] or list(CONFIGS))
