"""DETL v1 export (§8f-1): the GPU index serialises to exactly the bytes the
reference's save_index writes for the same build (persist.cpp:99-149), and the
reference's load_index accepts them and answers queries from them."""
import numpy as np
import pytest

from conftest import gaussian
from oracle.bindings import make_params

pytestmark = pytest.mark.gpu

CASES = [
    dict(n=20000, d=64, K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=50),
    dict(n=3000, d=16, K=8, L=2, n_regions=16, leaf_capacity=4, sample_fraction=0.5, beta=0.1, k=10),
]


@pytest.mark.parametrize("keep_codes", [True, False])
@pytest.mark.parametrize("case", CASES)
def test_save_index_bytes_equal_reference(gpu, ref, case, keep_codes):
    from paper_2406_10938_b200 import LshParams
    c = dict(case)
    n, d = c.pop("n"), c.pop("d")
    data = gaussian(n, d, n + d, 1.2)
    idx = gpu.build_index(data, LshParams(**c), seed=21, keep_codes=keep_codes)
    blob = idx.save_index()
    ri = ref.build_index(data, make_params(**c), 21)
    want = ri.save()
    assert len(blob) == len(want)
    assert blob == want
    # the reference loads the GPU-built index and answers from it
    li = ref.load_index(blob, data, make_params(**c))
    assert li is not None
    Q = gaussian(8, d, 5, 1.2)
    for q in Q:
        a = li.ck_ann(q, c["k"])
        b = ri.ck_ann(q, c["k"])
        assert len(a[0]) == len(b[0]) and a[3] == b[3]


def test_load_rejects_other_dataset(gpu, ref):
    from paper_2406_10938_b200 import LshParams
    c = dict(K=8, L=2, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.1, k=10)
    data = gaussian(2000, 12, 3, 1.0)
    blob = gpu.build_index(data, LshParams(**c), seed=2).save_index()
    other = data.copy()
    other[0, 0] += 1.0
    assert ref.load_index(blob, other, make_params(**c)) is None  # fingerprint mismatch
