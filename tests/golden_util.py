"""Loading of the reference-generated fixtures in tests/golden/ (see make_golden.py)."""
import glob
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))

from make_golden import CASES, make_data  # noqa: E402

FIELDS = ["K", "L", "c", "beta", "epsilon", "alpha1", "alpha2", "n_regions", "sample_fraction",
          "leaf_capacity", "r_min", "k"]


def cases():
    """The small fixtures of make_golden.py (the cfg_*.npz config fixtures of
    make_golden_configs.py are loaded by test_gpu_configs.py)."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "golden", "*.npz"))
                  if not os.path.basename(p).startswith("cfg_"))


def load(name):
    g = dict(np.load(os.path.join(HERE, "golden", f"{name}.npz")))
    kind, n, d, nq, pkw, seed, dseed = CASES[name]
    base, Q = make_data(kind, n, d, nq, dseed)
    return g, base, Q, pkw, seed


def tree_hash(t) -> str:
    return hashlib.sha256(np.ascontiguousarray(np.concatenate([
        t.root_children.view(np.uint8), t.is_leaf, t.split_dim, t.left.view(np.uint8),
        t.right.view(np.uint8), t.bits.ravel(), t.value.ravel(), t.ecount.view(np.uint8),
        t.positions.view(np.uint8)])).tobytes()).hexdigest()
