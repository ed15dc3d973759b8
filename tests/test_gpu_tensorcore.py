"""The tcgen05 (kind::i8) tile used for exact u8 verification: u8 x u8 -> s32
is exact, so the tile must equal the integer matrix product bit for bit."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N,K", [(256, 128), (32, 32), (128, 256), (64, 96)])
def test_tc_gemm_u8_exact(gpu, N, K):
    g = np.random.Generator(np.random.PCG64(N * 1000 + K))
    A = g.integers(0, 256, (128, K), dtype=np.uint8)
    B = g.integers(0, 256, (N, K), dtype=np.uint8)
    Cm = np.zeros((128, N), np.int32)
    rc = gpu.load().detlsh_test_tc_gemm_u8(C.c_void_p(A.ctypes.data), C.c_void_p(B.ctypes.data), N, K,
                                           C.c_void_p(Cm.ctypes.data))
    assert rc == 0, gpu.load().detlsh_gpu_last_error()
    want = A.astype(np.int64) @ B.astype(np.int64).T
    assert np.array_equal(Cm.astype(np.int64), want)


def _scopes(lib):
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
    return names.value.decode().split(";")[:m]


def _sparse_u8(g, n, d):
    return np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)


@pytest.mark.parametrize("d,k,nq,cap", [(128, 50, 5000, None), (100, 100, 600, None),
                                        (256, 20, 1500, None), (64, 30, 800, 120),
                                        (784, 50, 600, None), (300, 20, 700, None)])
def test_tc_verification_equals_gather_path_and_oracle(gpu, port, monkeypatch, d, k, nq, cap):
    """Dataset-major tcgen05 verification (u8 rows, budget >= 8192) returns the
    same (position, distance) lists as the per-query gather path and as the
    oracle, ties included (duplicated rows).  cap shrinks the survivor staging
    buffer so that queries overflow it and take the re-run."""
    from paper_2406_10938_b200 import LshParams
    if cap is not None:
        monkeypatch.setenv("DETLSH_TEST_TC_CAP", str(cap))
    g = np.random.Generator(np.random.PCG64(d * 7 + k))
    n = 120000
    data = _sparse_u8(g, n, d)
    data[n // 2: n // 2 + 500] = data[:500]  # exact duplicates -> distance ties
    Q = np.concatenate([_sparse_u8(g, nq - 100, d), data[g.integers(0, n, 100)]])
    Q[7] += 0.25  # non-integral -> fp64 gather path for this query
    c = dict(K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=k)
    idx = gpu.build_index(data, LshParams(**c), seed=11)
    assert idx.row_u8() % 32 == 0
    lib = gpu.load()
    lib.detlsh_profile_enable(1)
    ra = gpu.ck_ann_batch(idx, Q, k)
    lib.detlsh_profile_enable(0)
    assert "tc_score" in _scopes(lib), "tensor-core path not taken"
    rb = gpu.ck_ann_batch(idx, Q, k, tensor_cores=False)
    assert np.array_equal(ra.n_hits, rb.n_hits)
    assert np.array_equal(ra.ids, rb.ids)
    assert np.array_equal(ra.dists.view(np.uint64), rb.dists.view(np.uint64))
    assert np.array_equal(ra.candidates_seen, rb.candidates_seen)
    assert np.array_equal(ra.radius_used, rb.radius_used)
    from oracle.bindings import make_params
    oi = port.build_index(data, make_params(**c), 11)
    for qi in list(range(0, nq, max(1, nq // 12))) + [7, nq - 1]:
        ids, ds, rad, cs = oi.ck_ann(Q[qi], k)
        assert np.array_equal(ra.ids[qi], ids), f"query {qi}"
        assert np.array_equal(ra.dists[qi].view(np.uint64), np.asarray(ds).view(np.uint64)), f"query {qi}"
        assert ra.radius_used[qi] == rad and int(ra.candidates_seen[qi]) == cs


def test_host_buffers_pinned_and_pageable_agree(gpu):
    """The C-ABI query with pinned host buffers (direct copies) and with pageable
    ones (staged through the library's pinned buffers) returns the same bytes."""
    import ctypes as C
    import torch
    from paper_2406_10938_b200 import _lib
    rng = np.random.default_rng(5)
    data = rng.integers(0, 256, size=(20000, 64)).astype(np.float32)
    Q = rng.integers(0, 256, size=(300, 64)).astype(np.float32)
    idx = gpu.build_index(data, gpu.LshParams(beta=0.5, k=20), seed=3)
    ref = gpu.ck_ann_batch(idx, Q, 20)
    nq, k = Q.shape[0], 20
    qp = torch.from_numpy(Q).pin_memory()
    outs = [torch.zeros((nq, k), dtype=torch.int32).pin_memory(), torch.zeros((nq, k), dtype=torch.float64).pin_memory(),
            torch.zeros(nq, dtype=torch.int32).pin_memory(), torch.zeros(nq, dtype=torch.float64).pin_memory(),
            torch.zeros(nq, dtype=torch.int64).pin_memory()]
    p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    _lib.check(_lib.load().detlsh_gpu_query(idx.handle, p(qp), nq, k, 0, *[p(t) for t in outs], None))
    assert np.array_equal(outs[0].numpy().view(np.uint32), ref.ids)
    assert np.array_equal(outs[1].numpy().view(np.uint64), ref.dists.view(np.uint64))
    assert np.array_equal(outs[2].numpy(), ref.n_hits)
    assert np.array_equal(outs[3].numpy().view(np.uint64), ref.radius_used.view(np.uint64))
    assert np.array_equal(outs[4].numpy().view(np.uint64), ref.candidates_seen.view(np.uint64))


def _unit_gaussian(g, n, d):
    x = g.normal(0, 1, (n, d))
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


@pytest.mark.parametrize("kind,d,k,nq,cap", [("unit", 96, 50, 1500, None), ("mixture", 128, 50, 600, None),
                                             ("unit", 96, 20, 400, 100)])
def test_bf16x3_verification_equals_gather_path_and_oracle(gpu, port, monkeypatch, kind, d, k, nq, cap):
    """Float datasets: bf16-triple tcgen05 scores with a rigorous slack filter,
    survivors rescored in fp64 — the same (position, distance) lists as the
    fp64 gather path and the oracle (C4-like unit vectors; C1-like mixture
    with large norms; a tiny survivor cap forcing the gather re-run)."""
    from paper_2406_10938_b200 import LshParams
    if cap is not None:
        monkeypatch.setenv("DETLSH_TEST_TC_CAP", str(cap))
    g = np.random.Generator(np.random.PCG64(d * 13 + k))
    n = 120000
    if kind == "unit":
        data = _unit_gaussian(g, n + nq, d)
    else:
        centres = g.uniform(0, 100, (100, d))
        data = (centres[g.integers(0, 100, n + nq)] + g.normal(0, 5, (n + nq, d))).astype(np.float32)
    data, Q = np.ascontiguousarray(data[:n]), np.ascontiguousarray(data[n:])
    data[n // 2: n // 2 + 300] = data[:300]  # exact duplicates -> distance ties
    Q[:20] = data[g.integers(0, n, 20)]       # queries on data points (distance 0)
    c = dict(K=16, L=4, n_regions=256, leaf_capacity=128, sample_fraction=0.1, beta=0.1, k=k)
    idx = gpu.build_index(data, LshParams(**c), seed=5)
    assert idx.row_u8() == 0
    lib = gpu.load()
    lib.detlsh_profile_enable(1)
    ra = gpu.ck_ann_batch(idx, Q, k)
    lib.detlsh_profile_enable(0)
    assert "tc_score" in _scopes(lib), "bf16x3 tensor-core path not taken"
    rb = gpu.ck_ann_batch(idx, Q, k, tensor_cores=False)
    assert np.array_equal(ra.n_hits, rb.n_hits)
    assert np.array_equal(ra.ids, rb.ids)
    assert np.array_equal(ra.dists.view(np.uint64), rb.dists.view(np.uint64))
    assert np.array_equal(ra.candidates_seen, rb.candidates_seen)
    assert np.array_equal(ra.radius_used, rb.radius_used)
    from oracle.bindings import make_params
    oi = port.build_index(data, make_params(**c), 5)
    for qi in list(range(0, nq, max(1, nq // 10))) + [3, nq - 1]:
        ids, ds, rad, cs = oi.ck_ann(Q[qi], k)
        assert np.array_equal(ra.ids[qi], ids), f"query {qi}"
        assert np.array_equal(ra.dists[qi].view(np.uint64), np.asarray(ds).view(np.uint64)), f"query {qi}"
        assert ra.radius_used[qi] == rad and int(ra.candidates_seen[qi]) == cs
