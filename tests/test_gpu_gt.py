"""§8(f2): exact kNN ground truth on the GPU with brute_force_knn semantics
(metrics.cpp:8-33: sequential fp64 dist^2, (dist^2, position) order)."""
import numpy as np
import pytest

from conftest import gaussian, lattice

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,n,d,k", [("gauss", 20000, 48, 10), ("lattice", 5000, 12, 50),
                                         ("gauss", 3000, 200, 64), ("lattice", 700, 5, 700)])
def test_brute_force_knn_matches_oracle(gpu, port, kind, n, d, k):
    data = gaussian(n, d, n + d, 2.0) if kind == "gauss" else lattice(n, d, n + d, -2, 2)
    Q = np.concatenate([gaussian(40, d, 9, 2.0) if kind == "gauss" else lattice(40, d, 9, -2, 2), data[:7]])
    ids, ds = gpu.brute_force_knn(data, Q, k)
    oid, od = port.brute_force_knn(data, Q, k)
    assert np.array_equal(ids, oid)
    assert np.array_equal(ds.view(np.uint64), np.asarray(od).view(np.uint64))


def test_brute_force_knn_with_ann_bound(gpu, port):
    """The squared k-th ck_ann distance is a valid bound: same exact answer."""
    data = gaussian(30000, 32, 77, 1.0)
    Q = gaussian(64, 32, 78, 1.0)
    k = 20
    idx = gpu.build_index(data, gpu.LshParams(K=16, L=4, beta=0.1, k=k), seed=3)
    res = gpu.ck_ann_batch(idx, Q, k)
    bound = np.where(res.n_hits == k, res.dists[:, k - 1] ** 2 * (1 + 1e-12), np.inf)
    a = gpu.brute_force_knn(data, Q, k, dist2_bound=bound)
    b = gpu.brute_force_knn(data, Q, k)
    oid, od = port.brute_force_knn(data, Q, k)
    assert np.array_equal(a[0], oid) and np.array_equal(b[0], oid)
    assert np.array_equal(a[1], od) and np.array_equal(b[1], od)
