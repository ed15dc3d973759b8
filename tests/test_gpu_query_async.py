"""Stream-ordered batched ck_ann (include/detlsh_b200.h detlsh_gpu_query):
device-side overflow handling, no host waits, CUDA-graph capture."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sparse_u8(g, n, d):
    return np.where(g.random((n, d)) < 0.5, 0, np.minimum(g.geometric(0.05, (n, d)), 255)).astype(np.float32)


@pytest.fixture(scope="module")
def u8_index(gpu):
    g = np.random.Generator(np.random.PCG64(77))
    n, d = 60000, 128
    data = _sparse_u8(g, n, d)
    idx = gpu.build_index(data, gpu.LshParams(beta=0.2, k=20), seed=5)
    assert idx.row_u8() == 128
    return data, idx, g


def _far_queries(g, m, d):
    # far from every point: round 0 of tree 0 does not fill the budget, so
    # these queries take the general (slow) path
    return np.full((m, d), 255.0, np.float32) - g.integers(0, 3, (m, d)).astype(np.float32)


def test_pass_record_overflow_with_slow_queries(gpu, u8_index, monkeypatch):
    """A pass-record overflow in tc_score sends the whole chunk to the gather
    path on the device; more than half of the batch on the slow path must not
    overrun the slow-query list (each query is listed once)."""
    data, idx, g = u8_index
    k = 20
    Q = np.concatenate([_far_queries(g, 400, data.shape[1]), _sparse_u8(g, 200, data.shape[1])])
    want = gpu.ck_ann_batch(idx, Q, k, tensor_cores=False)
    assert (want.radius_used > idx.params.r_min).sum() > Q.shape[0] // 2, "slow path not exercised"
    monkeypatch.setenv("DETLSH_TEST_REC_CAP", "1000")
    got = gpu.ck_ann_batch(idx, Q, k)
    assert np.array_equal(got.n_hits, want.n_hits)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists.view(np.uint64), want.dists.view(np.uint64))
    assert np.array_equal(got.radius_used, want.radius_used)
    assert np.array_equal(got.candidates_seen, want.candidates_seen)


def test_small_batch_does_not_overflow_records(gpu, u8_index, monkeypatch):
    """rec_cap covers the runs the scorer's warps reserve ahead of use: a
    one-query batch on a u8 index must finish on the tensor-core path."""
    data, idx, g = u8_index
    Q = _sparse_u8(g, 1, data.shape[1])
    monkeypatch.setenv("DETLSH_TC_DEBUG", "1")
    want = gpu.ck_ann_batch(idx, Q, 20, tensor_cores=False)
    got = gpu.ck_ann_batch(idx, Q, 20)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists, want.dists)


def test_device_mode_is_stream_ordered_and_capturable(gpu, u8_index):
    """Device pointers: the call only enqueues (results appear after the stream
    is synchronised), two streams reuse the scratch in order, and after one
    warm-up call the enqueue can be captured into a CUDA graph and replayed."""
    import torch
    data, idx, g = u8_index
    k = 20
    Q = np.concatenate([_sparse_u8(g, 700, data.shape[1]), _far_queries(g, 20, data.shape[1])])
    want = gpu.ck_ann_batch(idx, Q, k)
    nq = Q.shape[0]
    dq = torch.from_numpy(Q).cuda()

    def outs():
        return (torch.full((nq, k), -1, dtype=torch.int32, device="cuda"),
                torch.zeros((nq, k), dtype=torch.float64, device="cuda"),
                torch.zeros(nq, dtype=torch.int32, device="cuda"),
                torch.zeros(nq, dtype=torch.float64, device="cuda"),
                torch.zeros(nq, dtype=torch.int64, device="cuda"))

    def same(o):
        m = want.n_hits
        assert np.array_equal(o[2].cpu().numpy(), m)
        assert np.array_equal(o[0].cpu().numpy().view(np.uint32), want.ids)
        assert np.array_equal(o[1].cpu().numpy().view(np.uint64), want.dists.view(np.uint64))
        assert np.array_equal(o[3].cpu().numpy(), want.radius_used)
        assert np.array_equal(o[4].cpu().numpy().view(np.uint64), want.candidates_seen)

    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    o1, o2 = outs(), outs()
    torch.cuda.synchronize()
    gpu.ck_ann_device(idx, dq, k, *o1, stream=s1.cuda_stream)
    gpu.ck_ann_device(idx, dq, k, *o2, stream=s2.cuda_stream)  # waits for s1's batch on the device
    torch.cuda.synchronize()
    same(o1)
    same(o2)
    gpu.query_check(idx)
    # graph capture of the (warm) enqueue, replayed twice into fresh outputs
    o3 = outs()
    s3 = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s3):
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=s3):
            gpu.ck_ann_device(idx, dq, k, *o3, stream=s3.cuda_stream)
    for _ in range(2):
        for t in o3:
            t.zero_()
        graph.replay()
        torch.cuda.synchronize()
        same(o3)


def _same(got, want):
    assert np.array_equal(got.n_hits, want.n_hits)
    assert np.array_equal(got.ids, want.ids)
    assert np.array_equal(got.dists.view(np.uint64), want.dists.view(np.uint64))
    assert np.array_equal(got.radius_used, want.radius_used)
    assert np.array_equal(got.candidates_seen, want.candidates_seen)


@pytest.mark.parametrize("k", [20, 1100])
def test_deferred_general_path(gpu, u8_index, monkeypatch, k):
    """With a large budget the general path defers the member distances to a
    grid-wide kernel and the top-k to one CTA per query (C5).  Forced here on
    a small index (DETLSH_SLOW_DEFER_MIN=0): far queries that need several
    rounds (count_within scored in the kernel) and, with k above the fast
    path's bound, a whole batch on the general path.  Results must equal the
    in-kernel general path bit for bit."""
    data, idx, g = u8_index
    d = data.shape[1]
    Q = np.concatenate([_far_queries(g, 24, d), _sparse_u8(g, 40, d)])
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", str(2**62))
    want = gpu.ck_ann_batch(idx, Q, k)
    assert (want.radius_used > idx.params.r_min).sum() >= 20, "multi-round general path not exercised"
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", "0")
    _same(gpu.ck_ann_batch(idx, Q, k), want)


def test_deferred_general_path_rc_ann(gpu, u8_index, monkeypatch):
    """rc_ann (a single pass; the c*r check on the k-th member) through the
    deferred general path equals the in-kernel one."""
    data, idx, g = u8_index
    d = data.shape[1]
    Q = np.concatenate([_far_queries(g, 8, d), _sparse_u8(g, 40, d)])
    r = idx.params.r_min
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", str(2**62))
    want = gpu.rc_ann_batch(idx, Q, r, 1.5)
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", "0")
    got = gpu.rc_ann_batch(idx, Q, r, 1.5)
    for a, b in zip(got, want):
        assert np.array_equal(np.asarray(a), np.asarray(b))


def test_general_path_after_budget_change(gpu, u8_index):
    """The budget (beta*n + k) lays out the general path's per-slot scratch; a
    batch with another k must not read an earlier batch's members as bitmap
    bits (the member bitmaps live apart and stay zero between queries)."""
    data, idx, g = u8_index
    d = data.shape[1]
    Q = np.concatenate([_far_queries(g, 24, d), _sparse_u8(g, 40, d)])
    first = gpu.ck_ann_batch(idx, Q, 600)
    gpu.ck_ann_batch(idx, Q, 1100)  # every query on the general path, larger budget
    _same(gpu.ck_ann_batch(idx, Q, 600), first)


@pytest.mark.parametrize("defer", [False, True])
def test_wide_ctas_equal(gpu, u8_index, monkeypatch, defer):
    """The C5 shapes (512-thread plan CTAs, 1024-thread general-path CTAs,
    chosen by index size) forced on a small index give the same results as
    the default 256-thread CTAs, with and without deferred member scoring."""
    data, idx, g = u8_index
    d = data.shape[1]
    Q = np.concatenate([_far_queries(g, 20, d), _sparse_u8(g, 300, d)])
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", "0" if defer else str(2**62))
    want = gpu.ck_ann_batch(idx, Q, 20)
    monkeypatch.setenv("DETLSH_FAST_THREADS", "512")
    monkeypatch.setenv("DETLSH_SLOW_THREADS", "1024")
    _same(gpu.ck_ann_batch(idx, Q, 20), want)
    _same(gpu.ck_ann_batch(idx, Q, 1100), gpu.ck_ann_batch(idx, Q, 1100, tensor_cores=False))


@pytest.mark.parametrize("defer", [False, True])
def test_general_path_u8_matches_oracle(gpu, port, monkeypatch, defer):
    """u8 index and u8-exact queries on the general path (integer member
    distances, in the kernel or deferred) equal the oracle bit for bit,
    including far queries that need several rounds."""
    from oracle.bindings import make_params
    g = np.random.Generator(np.random.PCG64(91))
    n, d, k = 20000, 64, 20
    data = _sparse_u8(g, n, d)
    idx = gpu.build_index(data, gpu.LshParams(beta=0.2, k=k), seed=5)
    oi = port.build_index(data, make_params(beta=0.2, k=k), 5)
    Q = np.concatenate([_far_queries(g, 12, d), _sparse_u8(g, 12, d)])
    monkeypatch.setenv("DETLSH_SLOW_DEFER_MIN", "0" if defer else str(2**62))
    monkeypatch.setenv("DETLSH_SLOW_THREADS", "1024" if defer else "256")
    res = gpu.ck_ann_batch(idx, Q, k)
    assert (res.radius_used > idx.params.r_min).sum() >= 10
    for qi in range(Q.shape[0]):
        ids, ds, rad, cs = oi.ck_ann(Q[qi], k)
        m = int(res.n_hits[qi])
        assert m == len(ids)
        assert np.array_equal(res.ids[qi, :m], ids), f"query {qi} ids"
        assert np.array_equal(res.dists[qi, :m].view(np.uint64), np.asarray(ds).view(np.uint64)), f"query {qi}"
        assert res.radius_used[qi] == rad
        assert int(res.candidates_seen[qi]) == cs


def test_batch_into_caller_arrays(gpu, u8_index):
    """ck_ann_batch(out=...) fills caller-owned (here page-locked) arrays with
    the same results, and rejects a wrongly typed one."""
    import torch
    data, idx, g = u8_index
    Q = _sparse_u8(g, 64, data.shape[1])
    want = gpu.ck_ann_batch(idx, Q, 20)
    pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()  # noqa: E731
    out = gpu.BatchResult(pin((64, 20), torch.int32).view(np.uint32), pin((64, 20), torch.float64),
                          pin((64,), torch.int32), pin((64,), torch.float64), pin((64,), torch.int64).view(np.uint64))
    got = gpu.ck_ann_batch(idx, Q, 20, out=out)
    assert got is out
    _same(got, want)
    bad = gpu.BatchResult(np.zeros((64, 20), np.int64), out.dists, out.n_hits, out.radius_used, out.candidates_seen)
    with pytest.raises(ValueError):
        gpu.ck_ann_batch(idx, Q, 20, out=bad)
