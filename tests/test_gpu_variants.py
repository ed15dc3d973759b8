"""§8(f4): the DET-ONLY (PAA) build variant and rc_ann, against the compiled
reference (build_det_only_index, index.cpp:220-232; rc_ann, index.cpp:267-290)."""
import numpy as np
import pytest

from conftest import gaussian, lattice
from oracle.bindings import make_params

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("case", [
    dict(n=20000, d=64, K=16, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=20),
    dict(n=3000, d=30, K=7, n_regions=16, leaf_capacity=8, sample_fraction=0.5, beta=0.1, k=10),
])
def test_det_only_index_matches_reference(gpu, ref, case):
    from paper_2406_10938_b200 import LshParams
    c = dict(case)
    n, d = c.pop("n"), c.pop("d")
    data = gaussian(n, d, n + 11, 1.0)
    idx = gpu.build_det_only_index(data, LshParams(**c), seed=4)
    ri = ref.build_det_only_index(data, make_params(**c), 4)
    assert idx.params.L == 1
    for f in ("epsilon", "alpha1", "alpha2", "beta", "r_min"):
        assert getattr(idx.params, f) == getattr(ri.params, f), f
    assert bits_equal(idx.table(), ri.table())
    assert idx.save_index() == ri.save()  # trees + projection kind + fingerprint
    Q = np.concatenate([gaussian(30, d, 12, 1.0), data[:: n // 10]])
    res = gpu.ck_ann_batch(idx, Q, c["k"])
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = ri.ck_ann(Q[qi], c["k"])
        m = int(res.n_hits[qi])
        assert np.array_equal(res.ids[qi, :m], ids), f"query {qi}"
        assert bits_equal(res.dists[qi, :m], ds), f"query {qi}"
        assert res.radius_used[qi] == rad and int(res.candidates_seen[qi]) == cs


@pytest.mark.parametrize("det_only", [False, True])
def test_rc_ann_matches_reference(gpu, ref, det_only):
    from paper_2406_10938_b200 import LshParams
    c = dict(K=12, n_regions=64, leaf_capacity=16, sample_fraction=0.2, beta=0.05, k=10)
    if not det_only:
        c["L"] = 3
    n, d = 8000, 24
    data = lattice(n, d, 31, -3, 3)  # integer lattice: distance ties
    if det_only:
        idx = gpu.build_det_only_index(data, LshParams(**c), seed=6)
        ri = ref.build_det_only_index(data, make_params(**c), 6)
    else:
        idx = gpu.build_index(data, LshParams(**c), seed=6)
        ri = ref.build_index(data, make_params(**c), 6)
    Q = np.concatenate([lattice(40, d, 32, -3, 3), data[:: n // 20]])
    for r in (0.5, 2.0, 4.0, 8.0):
        for cc in (1.2, 2.0):
            ids, ds, found, _ = gpu.rc_ann_batch(idx, Q, r, cc)
            for qi in range(Q.shape[0]):
                want = ri.rc_ann(Q[qi], r, cc)
                if want is None:
                    assert not found[qi], (r, cc, qi)
                else:
                    assert found[qi], (r, cc, qi)
                    assert int(ids[qi]) == want[0] and ds[qi] == want[1], (r, cc, qi)
    with pytest.raises(ValueError):
        gpu.rc_ann(idx, Q[0], 0.0, 2.0)
    with pytest.raises(ValueError):
        gpu.rc_ann(idx, Q[0], 1.0, 1.0)
