"""Reference entry points beyond build/ck_ann, through the C ABI, against the
compiled reference (oracle/_ref):

  estimate_rmin(index, probes, k)            index.hpp:91, index.cpp:333-374
  DetIndex::project_query(q, space)          index.cpp:181-188
  range_query_optimized(tree, table, q', r, sink)   de_tree.cpp:229-258
  range_query_exact(tree, table, q', r, lookup)     de_tree.cpp:199-227
"""
import numpy as np
import pytest

from oracle.bindings import make_params

pytestmark = pytest.mark.gpu

CASES = {
    "default": (dict(beta=0.1, k=10), "gauss", 20000, 24),
    "small": (dict(K=8, L=3, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.1, k=5), "lattice", 6000, 7),
}


def _data(kind, n, d, seed):
    g = np.random.Generator(np.random.PCG64(seed))
    if kind == "gauss":
        return g.normal(0, 2.0, (n, d)).astype(np.float32)
    return g.integers(-2, 3, (n, d)).astype(np.float32)


@pytest.fixture(scope="module", params=list(CASES))
def pair(request, ref):
    import paper_2406_10938_b200 as D
    pkw, kind, n, d = CASES[request.param]
    X = _data(kind, n + 40, d, 17)
    base, Q = X[:n], X[n:]
    gi = D.build_index(base, D.LshParams(**pkw), seed=21)
    ri = ref.build_index(base, make_params(**pkw), 21)
    assert gi.params.r_min == ri.params.r_min
    return gi, ri, base, Q, pkw


def test_project_query_matches_reference(pair):
    gi, ri, base, Q, pkw = pair
    P = gi.project_queries(Q)
    for i in range(gi.params.L):
        for q in range(Q.shape[0]):
            assert np.array_equal(P[i, q].view(np.uint32), ri.project_query(Q[q], i).view(np.uint32))


@pytest.mark.parametrize("np_,k", [(1, 1), (3, 10), (10, 50), (23, 7)])
def test_estimate_rmin_matches_reference(gpu, pair, np_, k):
    gi, ri, base, Q, pkw = pair
    probes = np.concatenate([Q, base[::97]])[:np_]
    got = gpu.estimate_rmin(gi, probes, k)
    want = ri.estimate_rmin(probes, k)
    assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64)


def test_estimate_rmin_rejects_empty_probes(gpu, pair):
    gi = pair[0]
    with pytest.raises(ValueError, match="no probe queries"):
        gpu.estimate_rmin(gi, np.zeros((0, gi.d()), np.float32), 5)


def test_range_queries_match_reference(gpu, pair):
    gi, ri, base, Q, pkw = pair
    eps, r_min = gi.params.epsilon, gi.params.r_min
    for tree in range(gi.params.L):
        P = gi.project_queries(Q[:6])[tree]
        for q in range(P.shape[0]):
            for scale in (0.5, 1.0, 2.25):
                radius = eps * r_min * scale
                for limit in (1, 37, 2**63):
                    got = gpu.range_query_optimized(gi, tree, P[q], radius, limit)
                    want = ri.range_query(tree, P[q], radius, limit)
                    assert np.array_equal(got, want), (tree, q, scale, limit)
                got = gpu.range_query_exact(gi, tree, P[q], radius)
                want = ri.range_query(tree, P[q], radius, exact=True)
                assert np.array_equal(got, want), (tree, q, scale, "exact")


def test_order_statistics_by_binning_equal_full_sort(gpu, monkeypatch):
    """Large samples take the boundary order statistics from a 16 K-bin
    monotone binning plus a sort of the wanted bins only; the table must equal
    the full sort's bit for bit, on rows with heavy duplicates, signed zeros,
    a constant row, a row holding +inf and a Gaussian row (n_s = 140 K)."""
    g = np.random.Generator(np.random.PCG64(11))
    L, n, K = 2, 700_000, 4
    pr = np.empty((L, n, K), np.float32)
    pr[0, :, 0] = g.standard_normal(n) * 3.0
    pr[0, :, 1] = g.integers(-3, 4, n).astype(np.float32)             # heavy duplicates
    pr[0, :, 2] = np.where(g.random(n) < 0.5, -0.0, 0.0) * (g.random(n) < 0.7) + (g.random(n) < 0.3) * g.standard_normal(n)
    pr[0, :, 3] = 1.25                                                 # constant
    pr[1, :, 0] = g.standard_normal(n).astype(np.float32)
    pr[1, :50, 0] = np.inf                                             # non-finite max
    pr[1, :, 1] = np.exp(g.standard_normal(n) * 6).astype(np.float32)  # wide dynamic range
    pr[1, :, 2] = -np.abs(g.standard_normal(n)).astype(np.float32)
    pr[1, :, 3] = (g.random(n) < 0.999) * 7.0
    for sample in ("gpu",):
        got = gpu.select_breakpoints(pr, 256, 0.2, 5, sample=sample)
        monkeypatch.setenv("DETLSH_TEST_FULL_ORDER_SORT", "1")
        want = gpu.select_breakpoints(pr, 256, 0.2, 5, sample=sample)
        monkeypatch.delenv("DETLSH_TEST_FULL_ORDER_SORT")
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), sample
