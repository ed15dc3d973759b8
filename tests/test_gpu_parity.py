"""GPU parity: every stage of the CUDA path against the CPU oracle on the same
seeded inputs, through the C ABI.  Bar: bit-exact (projections, breakpoints,
codes, trees incl. node order, r_min, result ids AND distances)."""
import numpy as np
import pytest

from conftest import gaussian, lattice
from oracle.bindings import make_params

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    if a.dtype.kind == "f":
        return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
    return a.shape == b.shape and np.array_equal(a, b)


def assert_tree_equal(t_gpu, t_orc, where=""):
    for f in ("root_children", "is_leaf", "split_dim", "left", "right", "bits", "value",
              "ebegin", "ecount", "positions"):
        g, o = getattr(t_gpu, f), getattr(t_orc, f)
        assert bits_equal(g, o), f"{where}: tree field {f} differs"


@pytest.mark.parametrize("n,d,K,L", [(1000, 128, 16, 4), (777, 5, 3, 2), (300, 1, 1, 1),
                                     (513, 130, 24, 3), (2049, 784, 16, 4), (64, 33, 7, 5)])
def test_project_dataset_bit_exact(gpu, port, n, d, K, L):
    data = gaussian(n, d, 11 + d, scale=3.0)
    fam = port.sample_hash_family(d, K, L, 99)
    np.testing.assert_array_equal(gpu.sample_hash_family(d, K, L, 99).view(np.uint32),
                                  fam.view(np.uint32))
    got = gpu.project_dataset(fam, data)
    want = port.project_dataset(fam, data)
    assert bits_equal(got, want)


@pytest.mark.parametrize("n,K,L,NR,frac", [(5000, 16, 4, 256, 0.1), (3000, 8, 4, 16, 0.5),
                                           (700, 3, 2, 8, 1.0), (260, 2, 3, 256, 0.9),
                                           (20000, 16, 4, 256, 0.1)])
def test_select_breakpoints_reference_sample(gpu, port, n, K, L, NR, frac):
    data = gaussian(n, 24, 5 + n, 2.0)
    if n == 700:
        data = np.round(data)  # duplicate-heavy sample
    fam = port.sample_hash_family(24, K, L, 3)
    proj = port.project_dataset(fam, data)
    want = port.select_breakpoints(proj, NR, frac, 1234)
    got = gpu.select_breakpoints(proj, NR, frac, 1234)
    assert bits_equal(got, want)


def test_select_breakpoints_gpu_sample_is_order_statistics(gpu, port):
    n, K, L, NR = 20000, 16, 4, 256
    proj = port.project_dataset(port.sample_hash_family(32, K, L, 4), gaussian(n, 32, 8))
    got = gpu.select_breakpoints(proj, NR, 0.1, 77, sample="gpu")
    assert np.all(np.diff(got, axis=2) >= 0)
    # every boundary is a value of its own projected coordinate
    for i in range(L):
        for j in range(K):
            col = set(proj[i, :, j].tolist())
            assert all(v in col for v in got[i, j, ::17].tolist())


@pytest.mark.parametrize("NR", [2, 16, 256])
def test_encode_dataset(gpu, port, NR):
    n, K, L = 4000, 16, 4
    proj = port.project_dataset(port.sample_hash_family(20, K, L, 9), gaussian(n, 20, 3))
    table = port.select_breakpoints(proj, NR, 0.2, 5)
    # plant boundary ties and out-of-range values
    proj = proj.copy()
    proj[0, :NR, 0] = table[0, 0, :NR]
    proj[1, 0, :] = -1e30
    proj[1, 1, :] = 1e30
    assert bits_equal(gpu.encode_dataset(proj, table), port.encode_dataset(proj, table))


@pytest.mark.parametrize("n,K,NR,leaf,kind", [(20000, 16, 256, 128, "gauss"),
                                              (3000, 8, 16, 16, "gauss"),
                                              (2000, 4, 8, 1, "gauss"),
                                              (1500, 3, 4, 8, "lattice"),
                                              (500, 1, 2, 3, "lattice"),
                                              (4000, 24, 256, 5, "gauss")])
def test_build_tree_matches_reference_insert_order(gpu, port, n, K, NR, leaf, kind):
    d = 12
    data = gaussian(n, d, n + K, 2.0) if kind == "gauss" else lattice(n, d, n + K, -1, 1)
    L = 2
    proj = port.project_dataset(port.sample_hash_family(d, K, L, 21), data)
    table = port.select_breakpoints(proj, NR, 0.5, 8)
    codes = port.encode_dataset(proj, table)
    for space in range(L):
        want = port.build_tree(codes, NR, space, leaf).export()
        got = gpu.build_tree(codes, space, leaf, NR)
        assert_tree_equal(got, want, f"space {space}")


def _params(**kw):
    from paper_2406_10938_b200 import LshParams
    return LshParams(**kw)


BUILD_CASES = [
    dict(n=5000, d=32, K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=10),
    dict(n=3000, d=16, K=8, L=4, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.1, k=10),
    dict(n=2000, d=16, K=8, L=4, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.01, k=5),
    dict(n=700, d=5, K=3, L=2, n_regions=8, leaf_capacity=2, sample_fraction=1.0, beta=0.1, k=10),
    dict(n=20000, d=64, K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.0, k=50),
]


@pytest.mark.parametrize("case", BUILD_CASES)
def test_build_index_and_queries(gpu, port, case):
    c = dict(case)
    n, d = c.pop("n"), c.pop("d")
    data = gaussian(n, d, n + d, 1.5)
    if n == 700:
        data = np.round(data)
    p = _params(**c)
    idx = gpu.build_index(data, p, seed=5)
    op = make_params(**c)
    oi = port.build_index(data, op, 5)
    # derived params, r_min, table, codes, trees
    for f in ("epsilon", "alpha1", "alpha2", "beta", "r_min"):
        assert getattr(idx.params, f) == getattr(oi.params, f), f
    assert bits_equal(idx.table(), oi.table())
    assert bits_equal(idx.family(), port.sample_hash_family(d, c["K"], c["L"], port.mix_seed(5, 0)))
    for i in range(c["L"]):
        assert_tree_equal(idx.tree(i), oi.tree_export(i), f"tree {i}")
    # queries: random + planted points
    Q = np.concatenate([gaussian(40, d, 77, 1.5), data[:: max(1, n // 10)][:10]])
    if n == 700:
        Q = np.round(Q)
    k = c["k"]
    res = gpu.ck_ann_batch(idx, Q, k)
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], k)
        m = int(res.n_hits[qi])
        assert m == len(ids)
        assert np.array_equal(res.ids[qi, :m], ids), f"query {qi} ids"
        assert bits_equal(res.dists[qi, :m], ds), f"query {qi} dists"
        assert res.radius_used[qi] == rad, f"query {qi} radius"
        assert int(res.candidates_seen[qi]) == cs, f"query {qi} candidates"


@pytest.mark.parametrize("L", [1, 3])
def test_reference_sample_with_zero_boundaries(gpu, port, L):
    """A third of the rows are all-zero, so many boundaries are exactly 0: the
    table rows come from GPU order statistics, and zero boundaries take the
    sign the reference's replayed quickselect leaves (incl. the last space,
    which is otherwise not replayed)."""
    n, d = 3000, 24
    data = gaussian(n, d, 41, 2.0)
    data[::3] = 0.0
    c = dict(K=8, L=L, n_regions=64, leaf_capacity=32, sample_fraction=0.3, beta=0.1, k=10)
    idx = gpu.build_index(data, _params(**c), seed=13)
    oi = port.build_index(data, make_params(**c), 13)
    t = np.asarray(idx.table())
    assert (t == 0.0).sum() > 0
    assert bits_equal(t, oi.table())
    for i in range(L):
        assert_tree_equal(idx.tree(i), oi.tree_export(i), f"tree {i}")


@pytest.mark.parametrize("borrow", [True, False])
def test_device_input_build_equals_host_input_build(gpu, borrow):
    """Reference-sample builds from a CUDA tensor (space 0's sample rows gathered
    on the device) and from host memory (gathered on the host, uploaded ahead of
    the dataset) give the same index."""
    import torch
    data = gaussian(6000, 48, 17, 2.0)
    c = dict(K=16, L=3, n_regions=256, leaf_capacity=64, sample_fraction=0.2, beta=0.1, k=10)
    a = gpu.build_index(data, _params(**c), seed=21)
    b = gpu.build_index(torch.from_numpy(data).cuda(), _params(**c), seed=21, borrow=borrow)
    assert bits_equal(a.table(), b.table())
    assert a.params.r_min == b.params.r_min
    for i in range(3):
        assert_tree_equal(a.tree(i), b.tree(i), f"tree {i}")


def test_exhaustive_budget_is_brute_force_with_ties(gpu, port):
    """beta = 1 (test_query.cpp:342-396): the pipeline reduces to exact kNN incl. tie order."""
    g = np.random.Generator(np.random.PCG64(401))
    for trial in range(12):
        n = int(2 + g.integers(0, 280))
        d = int(1 + g.integers(0, 12))
        discrete = trial % 2 == 0
        data = lattice(n, d, 500 + trial) if discrete else gaussian(n, d, 500 + trial, 2.0)
        regions = 2
        while regions * 2 <= 256 and regions * 2 <= n and g.integers(0, 2) == 0:
            regions *= 2
        p = _params(K=int(1 + g.integers(0, 8)), L=int(1 + g.integers(0, 3)), beta=1.0,
                    leaf_capacity=int(1 + g.integers(0, 8)), sample_fraction=1.0,
                    n_regions=regions)
        idx = gpu.build_index(data, p, seed=402 + trial)
        for k in (1, n // 2 + 1, n):
            q = lattice(1, d, 900 + trial)[0] if discrete else gaussian(1, d, 900 + trial, 2.0)[0]
            if k == 1:
                q = data[n // 2]
            r = gpu.ck_ann(idx, q, k)
            ids, ds = port.brute_force_knn(data, q[None], k)
            assert [h[0] for h in r.hits] == ids[0].tolist()
            assert np.array_equal(np.array([h[1] for h in r.hits]), ds[0])


def test_gpu_sample_mode_matches_hybrid_oracle(gpu, port):
    """GPU-native sample: everything downstream of the table equals the reference
    stage functions run with that same table (the hybrid oracle)."""
    n, d = 20000, 48
    data = gaussian(n, d, 42, 1.0)
    c = dict(K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=20)
    idx = gpu.build_index(data, _params(**c), seed=9, sample="gpu")
    table = idx.table()
    oi = port.build_index(data, make_params(**c), 9, table=table)
    assert idx.params.r_min == oi.params.r_min
    for i in range(4):
        assert_tree_equal(idx.tree(i), oi.tree_export(i), f"tree {i}")
    Q = gaussian(30, d, 43, 1.0)
    res = gpu.ck_ann_batch(idx, Q, 20)
    for qi in range(30):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], 20)
        assert np.array_equal(res.ids[qi], ids)
        assert bits_equal(res.dists[qi], ds)


def test_config2_subset_parity(gpu, port):
    from paper_2406_10938_b200 import data as gen
    base, Q = gen.make("c2", n=30000, nq=30)
    c = dict(K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=50)
    idx = gpu.build_index(base, _params(**c), seed=2)
    oi = port.build_index(base, make_params(**c), 2)
    assert idx.params.r_min == oi.params.r_min
    res = gpu.ck_ann_batch(idx, Q, 50)
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], 50)
        assert np.array_equal(res.ids[qi], ids)
        assert bits_equal(res.dists[qi], ds)
        assert res.radius_used[qi] == rad and int(res.candidates_seen[qi]) == cs


def test_errors_map_to_reference_taxonomy(gpu):
    data = gaussian(100, 8, 1)
    with pytest.raises(ValueError):
        gpu.build_index(data, _params(K=0))
    with pytest.raises(ValueError):
        gpu.build_index(data, _params(c=1.0))
    with pytest.raises(ValueError):
        gpu.build_index(data, _params(n_regions=256))  # sample too small for regions
    idx = gpu.build_index(data, _params(K=4, n_regions=8, sample_fraction=0.5, leaf_capacity=4), seed=1)
    with pytest.raises(ValueError):
        gpu.ck_ann(idx, np.zeros(7, np.float32), 5)
    with pytest.raises(ValueError):
        gpu.ck_ann(idx, np.zeros(8, np.float32), 0)
    with pytest.raises(ValueError):
        gpu.ck_ann(idx, np.zeros(8, np.float32), 101)


@pytest.mark.parametrize("d", [128, 20, 784 // 8])
def test_u8_rows_path_equals_fp64_path_and_oracle(gpu, port, d):
    """Integral datasets use exact int32 distances on u8 rows; both verification
    paths and the oracle must agree bit for bit, including a non-integral query
    (per-query fallback to the fp64 path)."""
    g = np.random.Generator(np.random.PCG64(d))
    n = 6000
    data = np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)
    Q = np.where(g.random((24, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (24, d)), 255)).astype(np.float32)
    Q[3] += 0.5  # not integral -> fp64 path for this query
    Q[5, 0] = 300.0  # out of u8 range -> fp64 path
    c = dict(K=16, L=4, n_regions=256, leaf_capacity=32, sample_fraction=0.1, beta=0.1, k=25)
    a = gpu.build_index(data, _params(**c), seed=4)
    b = gpu.build_index(data, _params(**c), seed=4, u8_rows=False)
    ra, rb = gpu.ck_ann_batch(a, Q, 25), gpu.ck_ann_batch(b, Q, 25)
    assert np.array_equal(ra.ids, rb.ids) and bits_equal(ra.dists, rb.dists)
    oi = port.build_index(data, make_params(**c), 4)
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], 25)
        assert np.array_equal(ra.ids[qi], ids) and bits_equal(ra.dists[qi], ds)


@pytest.mark.parametrize("case", [
    dict(n=20000, d=64, K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=50),
    dict(n=6000, d=24, K=12, L=2, n_regions=64, leaf_capacity=8, sample_fraction=0.5, beta=0.1, k=20),
])
def test_approximate_leaf_scan_equals_exact_scan(gpu, monkeypatch, case):
    """The fp32 leaf scan (half-code tables, refined dims, margin classification)
    must select exactly the leaves the all-fp64 scan selects."""
    c = dict(case)
    n, d = c.pop("n"), c.pop("d")
    data = gaussian(n, d, n + 3, 1.3)
    idx = gpu.build_index(data, _params(**c), seed=8)
    Q = np.concatenate([gaussian(300, d, 9, 1.3), data[:: n // 50]])
    ra = gpu.ck_ann_batch(idx, Q, c["k"])
    monkeypatch.setenv("DETLSH_TEST_EXACT_SCAN", "1")
    rb = gpu.ck_ann_batch(idx, Q, c["k"])
    assert np.array_equal(ra.ids, rb.ids)
    assert bits_equal(ra.dists, rb.dists)
    assert np.array_equal(ra.candidates_seen, rb.candidates_seen)


@pytest.mark.parametrize("case", [
    dict(n=3000, d=16, K=20, L=2, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.1, k=10),
    dict(n=100, d=8, K=6, L=2, n_regions=8, leaf_capacity=128, sample_fraction=1.0, beta=0.5, k=5),
])
def test_query_paths_without_half_form(gpu, port, case):
    """K > 16 (no approximate scan) and a root-leaf tree (no half form) match the oracle."""
    c = dict(case)
    n, d = c.pop("n"), c.pop("d")
    data = gaussian(n, d, n + 5, 1.0)
    idx = gpu.build_index(data, _params(**c), seed=3)
    oi = port.build_index(data, make_params(**c), 3)
    Q = gaussian(20, d, 6, 1.0)
    res = gpu.ck_ann_batch(idx, Q, c["k"])
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], c["k"])
        m = int(res.n_hits[qi])
        assert np.array_equal(res.ids[qi, :m], ids), f"query {qi}"
        assert bits_equal(res.dists[qi, :m], ds), f"query {qi}"
