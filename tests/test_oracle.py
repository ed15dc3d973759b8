"""The CPU oracle pinned against the reference's own golden values, known-answer
tests and fixtures, and — when oracle/_ref is built — against the
reference library itself, bit for bit, on seeded inputs."""
import math

import numpy as np
import pytest

from conftest import gaussian, lattice
from golden_util import FIELDS, cases, load, tree_hash
from oracle.bindings import make_params


def test_derived_params_golden(port):
    # test_cli.cpp:60-61 (alpha1 0.7788007831, beta 0.0379945254) and SURVEY §8a3
    p = port.derive_params(16, 1.5, 4)
    assert f"{p['alpha1']:.10f}" == "0.7788007831"
    assert f"{p['beta']:.10f}" == "0.0379945254"
    assert f"{p['epsilon']:.10f}" == "3.3885146991"
    assert f"{p['alpha2']:.10f}" == "0.9952164704"


def test_chi2_closed_forms(port):
    # test_projection.cpp:13-21: k=2 closed forms
    for a in (0.05, 0.3, 0.7788007831, 0.99):
        assert abs(port.chi2_quantile(a, 2) + 2.0 * math.log(a)) <= 1e-9
    for x in (0.1, 1.0, 5.0, 20.0):
        assert abs(port.chi2_cdf(x, 2) - (1.0 - math.exp(-x / 2))) <= 1e-12
    assert port.chi2_quantile(1.0, 5) == 0.0


def test_candidate_budget_golden(port):
    # test_query.cpp:36-41
    assert port.candidate_budget(0.1, 1000, 5) == 105
    assert port.candidate_budget(0.1, 14, 1) == 3
    assert port.candidate_budget(0.5, 10, 50) == 10
    assert port.candidate_budget(0.0, 10, 3) == 3


def test_breakpoint_hand_rows_and_sort_oracle(port):
    # test_encoder.cpp:13-59 / test_util.hpp:69-78: interior boundary t at sorted
    # rank floor(n_s/N_r)*t - 1, ends at the sample extremes; duplicates too.
    g = np.random.Generator(np.random.PCG64(3))
    for trial in range(40):
        n_regions = [2, 4, 16, 256][trial % 4]
        n_s = int(n_regions + g.integers(0, 3000))
        s = (g.integers(-5, 6, n_s) if trial % 3 == 0 else g.normal(0, 1, n_s)).astype(np.float32)
        row, _ = port.select_row_breakpoints(s, n_regions, 1000 + trial)
        srt = np.sort(s)
        span = n_s // n_regions
        want = np.empty(n_regions + 1, np.float32)
        want[0], want[-1] = srt[0], srt[-1]
        for t in range(1, n_regions):
            want[t] = srt[span * t - 1]
        assert np.array_equal(row, want)


def test_locate_region_ties_and_clamps(port):
    # test_encoder.cpp:83-91
    row = np.array([0, 1, 2, 3, 4], np.float32)  # 4 regions
    assert port.locate_region(-1.0, row) == 0
    assert port.locate_region(0.0, row) == 0  # the global minimum maps to region 0
    assert port.locate_region(1.0, row) == 0  # boundary tie -> lower region
    assert port.locate_region(1.5, row) == 1
    assert port.locate_region(4.0, row) == 3
    assert port.locate_region(9.0, row) == 3


@pytest.mark.parametrize("name", cases())
def test_oracle_reproduces_reference_fixtures(port, name):
    g, base, Q, pkw, seed = load(name)
    idx = port.build_index(base, make_params(**pkw), seed)
    got = [getattr(idx.params, f) for f in FIELDS]
    assert np.array_equal(np.array(got, np.float64), g["params"])
    assert np.array_equal(idx.table().view(np.uint32), g["table"].view(np.uint32))
    for i in range(int(g["params"][1])):
        assert tree_hash(idx.tree_export(i)) == str(g["tree_hash"][i])
    k = int(g["params"][11])
    for i in range(Q.shape[0]):
        ids, ds, rad, cs = idx.ck_ann(Q[i], k)
        m = int(g["n_hits"][i])
        assert np.array_equal(ids, g["ids"][i, :m])
        assert np.array_equal(ds, g["dists"][i, :m])
        assert rad == g["radius"][i] and cs == g["cands"][i]


@pytest.mark.parametrize("n,d,K,L,NR,leaf,frac,disc", [
    (5000, 32, 16, 4, 256, 128, 0.1, False), (3000, 16, 8, 4, 16, 16, 0.5, False),
    (700, 5, 3, 2, 8, 2, 1.0, True), (1200, 7, 24, 2, 256, 3, 0.5, False),
    (300, 2, 1, 3, 4, 1, 1.0, True)])
def test_oracle_matches_reference_library(port, ref, n, d, K, L, NR, leaf, frac, disc):
    data = lattice(n, d, n) if disc else gaussian(n, d, n, 2.0)
    fam = port.sample_hash_family(d, K, L, 77)
    assert np.array_equal(fam.view(np.uint32), ref.sample_hash_family(d, K, L, 77).view(np.uint32))
    pr = port.project_dataset(fam, data)
    assert np.array_equal(pr.view(np.uint32), ref.project_dataset(fam, data).view(np.uint32))
    t1 = port.select_breakpoints(pr, NR, frac, 99)
    assert np.array_equal(t1.view(np.uint32), ref.select_breakpoints(pr, NR, frac, 99).view(np.uint32))
    c1 = port.encode_dataset(pr, t1)
    assert np.array_equal(c1, ref.encode_dataset(pr, t1))
    for sp in range(L):
        assert tree_hash(port.build_tree(c1, NR, sp, leaf).export()) == \
            tree_hash(ref.build_tree(c1, NR, sp, leaf).export())
    p = make_params(K=K, L=L, n_regions=NR, leaf_capacity=leaf, sample_fraction=frac, beta=0.1, k=5)
    i1, i2 = port.build_index(data, p, 5), ref.build_index(data, p, 5)
    assert i1.params.r_min == i2.params.r_min
    for q in gaussian(10, d, 3, 2.0):
        a, b = i1.ck_ann(q, 5), i2.ck_ann(q, 5)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2:] == b[2:]


def test_rng_streams_match_reference(port, ref):
    for seed in (0, 1, 12345, 2**63 + 7):
        u1, g1 = port.rng_stream(seed, 2000)
        u2, g2 = ref.rng_stream(seed, 2000)
        assert np.array_equal(u1, u2) and np.array_equal(g1.view(np.uint64), g2.view(np.uint64))
        assert port.mix_seed(seed, 3) == ref.mix_seed(seed, 3)


def test_port_reproduces_full_c1_fixture(port):
    """The C restatement against the reference's full-size C1 result
    (tests/golden/cfg_c1.npz, made by the compiled reference): same table,
    trees, r_min and answers on a strided third of the 1,000 queries."""
    import os
    from golden_util import FIELDS
    from paper_2406_10938_b200 import data as gen
    g = dict(np.load(os.path.join(os.path.dirname(__file__), "golden", "cfg_c1.npz")))
    base, Q = gen.make("c1")
    idx = port.build_index(base, make_params(beta=0.1, k=50), int(g["seed"]))
    got = np.array([getattr(idx.params, f) for f in FIELDS], np.float64)
    assert np.array_equal(got.view(np.uint64), g["params"].view(np.uint64))
    assert np.array_equal(idx.table().view(np.uint32), g["table"].view(np.uint32))
    for i in range(4):
        assert tree_hash(idx.tree_export(i)) == str(g["tree_hash"][i])
    for i in range(0, int(g["nq"]), 3):
        ids, ds, rad, cs = idx.ck_ann(Q[i], 50)
        m = int(g["n_hits"][i])
        assert np.array_equal(ids, g["ids"][i, :m]) and np.array_equal(ds, g["dists"][i, :m])
        assert rad == g["radius"][i] and cs == g["cands"][i]
