"""CPU-side checks of the product library: it loads, exports every symbol the
C header declares, its host determinism core equals the oracle, and argument
validation raises the reference's exception kinds before touching a device."""
import ctypes

import numpy as np
import pytest

import paper_2406_10938_b200 as D


def test_library_exports_every_header_symbol():
    lib = D.load()
    syms = D.header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s


def test_no_cpu_fallback_when_library_missing(monkeypatch, tmp_path):
    from paper_2406_10938_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    with pytest.raises(ImportError):
        _lib.load()


def test_host_numerics_match_oracle(port):
    for K, c, L in [(16, 1.5, 4), (8, 1.5, 4), (1, 2.0, 1), (24, 1.2, 7)]:
        a = D.derive_params(K, c, L)
        b = port.derive_params(K, c, L)
        assert (a.alpha1, a.alpha2, a.epsilon, a.beta) == (b["alpha1"], b["alpha2"], b["epsilon"], b["beta"])
    for beta, n, k in [(0.1, 1000, 5), (0.1, 14, 1), (0.5, 10, 50), (0.0, 10, 3), (0.1, 10**6, 50)]:
        assert D.candidate_budget(beta, n, k) == port.candidate_budget(beta, n, k)
    for seed in (0, 3, 2**40 + 1):
        for s in range(3):
            assert D.mix_seed(seed, s) == port.mix_seed(seed, s)
    for d, K, L in [(128, 16, 4), (5, 3, 2), (784, 16, 4)]:
        seed = port.mix_seed(7, 0)
        assert np.array_equal(D.sample_hash_family(d, K, L, seed).view(np.uint32),
                              port.sample_hash_family(d, K, L, seed).view(np.uint32))
    for x, k in [(3.0, 16), (0.5, 1), (40.0, 24)]:
        assert D.chi2_cdf(x, k) == port.chi2_cdf(x, k)
        assert D.chi2_quantile(0.3, k) == port.chi2_quantile(0.3, k)


def test_validation_is_invalid_argument_without_gpu():
    data = np.zeros((100, 8), np.float32)
    for kw in [dict(K=0), dict(K=25), dict(L=0), dict(c=1.0), dict(leaf_capacity=0),
               dict(n_regions=3), dict(n_regions=512), dict(sample_fraction=0.0),
               dict(sample_fraction=1.5), dict(n_regions=256)]:
        with pytest.raises(ValueError):
            D.build_index(data, D.LshParams(**kw))
    with pytest.raises(ValueError):
        D.build_index(np.zeros((0, 8), np.float32))


def test_params_struct_layout_matches_header():
    # detlsh_params: int32 K, L; 5 doubles; int32; double; int32; double; int32
    assert ctypes.sizeof(D._lib.Params) == 88
    assert D._lib.Params.r_min.offset == 72


def _select_row(sample, n_regions, seed):
    s = np.array(sample, np.float32)
    row = np.empty(n_regions + 1, np.float32)
    dr = ctypes.c_uint64(0)
    D._lib.check(D.load().detlsh_select_row_breakpoints(
        ctypes.c_void_p(s.ctypes.data), len(s), n_regions, seed,
        ctypes.c_void_p(row.ctypes.data), ctypes.byref(dr)))
    return row, s, dr.value


@pytest.mark.parametrize("trial", range(72))
def test_host_replay_matches_oracle_partition_for_partition(port, trial):
    """The blocked Hoare scan, and the closed-form rewrite taken when the pivot
    value is unique in its segment, reproduce the reference's sentinel loop
    exactly: same boundaries AND the same final arrangement (so the same later
    pivots)."""
    g = np.random.Generator(np.random.PCG64(100 + trial))
    n_regions = [2, 8, 16, 256][trial % 4]
    n_s = int(n_regions + g.integers(0, [500, 5000, 60000][trial % 3]))
    kind = trial % 6
    if kind == 0:
        s = g.normal(0, 1, n_s)
    elif kind == 1:
        s = g.integers(-3, 4, n_s)  # heavy duplicates
    elif kind == 2:
        s = np.sort(g.normal(0, 1, n_s))  # presorted
    elif kind == 3:
        s = np.full(n_s, 2.5)  # all equal
    elif kind == 4:
        s = np.sort(g.normal(0, 1, n_s))[::-1]  # reversed
    else:  # distinct values with a block of signed zeros (pivot ties on -0 == +0)
        s = g.normal(0, 1, n_s)
        z = g.random(n_s) < 0.3
        s[z] = np.where(g.random(int(z.sum())) < 0.5, -0.0, 0.0)
    s = s.astype(np.float32)
    row, arr, draws = _select_row(s, n_regions, 77 + trial)
    orow, oarr = port.select_row_breakpoints(s, n_regions, 77 + trial)
    assert np.array_equal(row.view(np.uint32), orow.view(np.uint32))
    assert np.array_equal(arr.view(np.uint32), oarr.view(np.uint32))
    assert draws > 0 or n_s <= 8
