"""Tensor-core projection of 8-bit-integer data (csrc/project_tc.cu) against
the oracle's project_dataset (projection.cpp:31-37): bit-exact, including the
certified-rounding fixup list, the guarded FP64 fallback (cap overflow and
non-integral data) and shapes off the fast path's sweet spot."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_2406_10938_b200 import data as gen

pytestmark = pytest.mark.gpu


def profiled(gpu, fn):
    lib = gpu.load()
    lib.detlsh_profile_enable(1)
    out = fn()
    lib.detlsh_profile_enable(0)
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
    return out, set(names.value.decode().split(";")[:m])


def u8_data(n, d, seed, zero_frac=0.5):
    g = np.random.Generator(np.random.PCG64(seed))
    x = np.minimum(255, g.geometric(0.05, (n, d)) - 1).astype(np.float32)
    x[g.random((n, d)) < zero_frac] = 0
    return x


@pytest.mark.parametrize("n,d,K,L", [(20000, 128, 16, 4), (9000, 100, 16, 4), (8192, 96, 24, 4),
                                     (20000, 192, 16, 4), (5000, 20, 16, 1), (4100, 64, 7, 3)])
def test_tc_projection_bit_exact(gpu, port, n, d, K, L):
    data = u8_data(n, d, 3 + d)
    fam = port.sample_hash_family(d, K, L, 17 + K)
    got, scopes = profiled(gpu, lambda: gpu.project_dataset(fam, data))
    assert "project_tc" in scopes, scopes
    want = port.project_dataset(fam, data)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_wide_rows_fall_back_exactly(gpu, port):
    """d = 256: the staging ring no longer holds a whole tile, so the launch
    takes the FP64 DMMA kernel; same bits either way."""
    data = u8_data(20000, 256, 9)
    fam = port.sample_hash_family(256, 16, 4, 31)
    got, scopes = profiled(gpu, lambda: gpu.project_dataset(fam, data))
    assert "project_tc" not in scopes
    assert np.array_equal(got.view(np.uint32), port.project_dataset(fam, data).view(np.uint32))


def test_tc_projection_c2_rows(gpu, port):
    base, _ = gen.make("c2", n=30000, nq=0)
    fam = port.sample_hash_family(128, 16, 4, 5)
    got = gpu.project_dataset(fam, base)
    assert np.array_equal(got.view(np.uint32), port.project_dataset(fam, base).view(np.uint32))


@pytest.mark.parametrize("mode", ["fixups", "overflow", "nonintegral", "dense255"])
def test_tc_projection_fallbacks(gpu, port, mode, monkeypatch, capfd):
    n, d, K, L = 8192, 128, 16, 4
    data = u8_data(n, d, 77, zero_frac=0.0 if mode == "dense255" else 0.5)
    if mode == "dense255":
        data[:] = 255.0
        data[::7, ::3] = 0.0
    if mode == "fixups":  # widen the band: thousands of outputs go to the fp64 fixup list
        monkeypatch.setenv("DETLSH_TEST_PROJ_ERR_SCALE", "2048")
    if mode == "overflow":  # list too small: the guarded DMMA kernel recomputes everything
        monkeypatch.setenv("DETLSH_TEST_PROJ_CAP", "0")
        monkeypatch.setenv("DETLSH_TEST_PROJ_ERR_SCALE", "64")
    if mode == "nonintegral":
        data[4321, 17] = 0.5
    fam = port.sample_hash_family(d, K, L, 23)
    monkeypatch.setenv("DETLSH_DEBUG_PROJ", "1")
    capfd.readouterr()
    got, scopes = profiled(gpu, lambda: gpu.project_dataset(fam, data))
    assert "project_tc" in scopes and "project_fixup" in scopes
    line = [x for x in capfd.readouterr().err.splitlines() if x.startswith("[project_tc]")][-1]
    kv = dict(t.split("=") for t in line.split()[1:])
    undecided, cap = int(kv["undecided"]), int(kv["cap"])
    assert int(kv["nonintegral"]) == (mode == "nonintegral")
    if mode == "fixups":
        assert 1000 < undecided <= cap, line  # the fp64 fixup list, not the full DMMA rerun
    if mode == "overflow":
        assert undecided > cap == 0, line
    want = port.project_dataset(fam, data)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_tc_projection_in_index_build(gpu, port):
    """The index build projects with the tensor-core kernel; the whole build
    (table, codes, trees, r_min) still matches the oracle."""
    from oracle.bindings import make_params
    base, Q = gen.make("c2", n=20000, nq=8)
    p = gpu.LshParams(beta=0.1, k=10)
    (idx, scopes) = profiled(gpu, lambda: gpu.build_index(base, p, seed=2, device=0))
    assert "project_tc" in scopes, scopes
    oi = port.build_index(base, make_params(beta=0.1, k=10), 2)
    assert idx.params.r_min == oi.params.r_min
    assert np.array_equal(idx.table().view(np.uint32), oi.table().view(np.uint32))
    res = gpu.ck_ann_batch(idx, Q, 10)
    for i in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[i], 10)
        assert np.array_equal(res.ids[i, :len(ids)], ids)
        assert np.array_equal(res.dists[i, :len(ds)], ds)
