"""Generate the golden fixtures in tests/golden/ from the REAL reference
(oracle/_ref/libdetlsh_ref.so, built from /root/reference/proj/src by
`make -C oracle ref`).  Run in the dev container:

    python tests/golden/make_golden.py

Each fixture pins a small seeded workload: the inputs are regenerated from
the recorded seeds (numpy PCG64), the outputs are the reference's.
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.bindings import Oracle, make_params  # noqa: E402

CASES = {
    # name: (data kind, n, d, nq, params, seed, data_seed)
    "gauss_small": ("gauss", 3000, 16, 12, dict(K=8, L=4, n_regions=16, leaf_capacity=16,
                                                 sample_fraction=0.5, beta=0.1, k=10), 152, 151),
    "gauss_default": ("gauss", 6000, 32, 12, dict(beta=0.1, k=50), 5, 42),
    "lattice_tiny": ("lattice", 400, 5, 8, dict(K=3, L=2, n_regions=8, leaf_capacity=2,
                                                sample_fraction=1.0, beta=0.2, k=7), 7, 9),
    "c2_subset": ("c2", 20000, 128, 10, dict(beta=0.1, k=50), 2, 2),
}


def make_data(kind, n, d, nq, data_seed):
    g = np.random.Generator(np.random.PCG64(data_seed))
    if kind == "gauss":
        allp = g.normal(0, 1.5, (n + nq, d)).astype(np.float32)
    elif kind == "lattice":
        allp = g.integers(-2, 3, (n + nq, d)).astype(np.float32)
    else:
        from paper_2406_10938_b200 import data as gen
        return gen.make("c2", n=n, nq=nq)
    return allp[:n], allp[n:]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    ref = Oracle("reference")
    for name, (kind, n, d, nq, pkw, seed, dseed) in CASES.items():
        base, Q = make_data(kind, n, d, nq, dseed)
        p = make_params(**pkw)
        idx = ref.build_index(base, p, seed)
        k = pkw["k"]
        ids = np.zeros((nq, k), np.uint32)
        ds = np.zeros((nq, k), np.float64)
        rad = np.zeros(nq)
        cs = np.zeros(nq, np.uint64)
        nh = np.zeros(nq, np.int32)
        for i in range(nq):
            a, b, r, c = idx.ck_ann(Q[i], k)
            ids[i, :len(a)], ds[i, :len(a)], rad[i], cs[i], nh[i] = a, b, r, c, len(a)
        p = idx.params
        trees = [idx.tree_export(i) for i in range(p.L)]
        out = dict(
            kind=kind, n=n, d=d, nq=nq, seed=seed, data_seed=dseed,
            params=np.array([p.K, p.L, p.c, p.beta, p.epsilon, p.alpha1, p.alpha2, p.n_regions,
                             p.sample_fraction, p.leaf_capacity, p.r_min, p.k], np.float64),
            table=idx.table(), ids=ids, dists=ds, radius=rad, cands=cs, n_hits=nh,
            tree_nodes=np.array([len(t.is_leaf) for t in trees]),
            tree_hash=np.array([sha(np.concatenate([t.root_children.view(np.uint8), t.is_leaf,
                                                    t.split_dim, t.left.view(np.uint8),
                                                    t.right.view(np.uint8), t.bits.ravel(),
                                                    t.value.ravel(), t.ecount.view(np.uint8),
                                                    t.positions.view(np.uint8)]))
                                for t in trees]),
        )
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print(name, "r_min", p.r_min, "nodes", out["tree_nodes"].tolist())


if __name__ == "__main__":
    main()
