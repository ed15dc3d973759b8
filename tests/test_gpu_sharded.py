"""The single-process point-sharded C-ABI (detlsh_gpu_sharded_*):
several shards on device 0 stand in for one shard per GPU (the code path is
the same: per-shard streams, peer copies to the merge device, merge kernel).
Parity: the reference algorithm (oracle port) run on each shard, then the
merge by (distance, global position)."""
import numpy as np
import pytest

from oracle.bindings import make_params
from test_sharding import merge_reference

pytestmark = pytest.mark.gpu


def _shard_oracle(port, base, Q, shards, pkw, seed, k):
    n = base.shape[0]
    nq = Q.shape[0]
    d = np.zeros((shards, nq, k))
    i = np.zeros((shards, nq, k), np.int64)
    h = np.zeros((shards, nq), np.int32)
    idxs = []
    for s in range(shards):
        s0, s1 = s * n // shards, (s + 1) * n // shards
        idx = port.build_index(base[s0:s1], make_params(**pkw), seed)
        idxs.append(idx)
        for q in range(nq):
            ids, ds, _, _ = idx.ck_ann(Q[q], k)
            d[s, q, :len(ids)], i[s, q, :len(ids)], h[s, q] = ds, ids.astype(np.int64) + s0, len(ids)
    return merge_reference(d, i, h, k), idxs


@pytest.mark.parametrize("shards,u8", [(2, False), (3, True)])
def test_sharded_build_and_query_match_per_shard_oracle(gpu, port, shards, u8):
    g = np.random.Generator(np.random.PCG64(31 + shards))
    n, dim, nq, k = 24001, 32, 40, 10
    if u8:
        base = np.where(g.random((n + nq, dim)) < 0.5, 0, np.minimum(g.geometric(0.05, (n + nq, dim)), 255))
        base = base.astype(np.float32)
    else:
        base = g.normal(0, 2.0, (n + nq, dim)).astype(np.float32)
    base, Q = base[:n], base[n:]
    pkw = dict(beta=0.1, k=k)
    sx = gpu.build_sharded_index(base, gpu.LshParams(**pkw), seed=9, devices=[0] * shards)
    assert sx.shard_count() == shards
    (od, oi, oh), oidx = _shard_oracle(port, base, Q, shards, pkw, 9, k)
    for s in range(shards):
        v = sx.shard(s)
        assert v.rows == (s * n // shards, (s + 1) * n // shards)
        assert v.params.r_min == oidx[s].params.r_min
        assert np.array_equal(v.table().view(np.uint32), oidx[s].table().view(np.uint32))
    ids, ds, nh = gpu.ck_ann_sharded(sx, Q, k)
    assert np.array_equal(nh, oh)
    assert np.array_equal(ids.astype(np.int64), oi)
    assert np.array_equal(ds, od)


def test_sharded_device_mode_matches_host_mode(gpu):
    import torch
    g = np.random.Generator(np.random.PCG64(8))
    n, dim, nq, k = 40000, 64, 300, 20
    base = g.integers(0, 256, (n, dim)).astype(np.float32)
    Q = g.integers(0, 256, (nq, dim)).astype(np.float32)
    sx = gpu.build_sharded_index(base, gpu.LshParams(beta=0.3, k=k), seed=4, devices=[0, 0, 0, 0])
    hi, hd, hh = gpu.ck_ann_sharded(sx, Q, k)
    dq = torch.from_numpy(Q).cuda()
    ids = torch.zeros((nq, k), dtype=torch.int64, device="cuda")
    ds = torch.zeros((nq, k), dtype=torch.float64, device="cuda")
    nh = torch.zeros(nq, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()
    gpu.ck_ann_sharded_device(sx, dq, k, ids, ds, nh, stream=s.cuda_stream)
    torch.cuda.synchronize()
    assert np.array_equal(nh.cpu().numpy(), hh)
    assert np.array_equal(ids.cpu().numpy().view(np.uint64), hi)
    assert np.array_equal(ds.cpu().numpy(), hd)
    # the shards answer like single indexes over their rows
    for sidx in range(4):
        v = sx.shard(sidx)
        r = gpu.ck_ann_batch(v, Q[:5], k)
        assert r.n_hits.min() == k


def test_merge_topk_many_shards(gpu):
    """The warp-per-query merge has no 16-shard cap (here 40 shards)."""
    import torch
    g = np.random.Generator(np.random.PCG64(12))
    S, nq, k = 40, 64, 8
    d = np.sort(g.integers(0, 30, (S, nq, k)).astype(np.float64), axis=2)
    ids = g.permutation(S * nq * k).reshape(S, nq, k).astype(np.int64)
    hits = g.integers(0, k + 1, (S, nq)).astype(np.int32)
    for s in range(S):
        for q in range(nq):
            o = np.lexsort((ids[s, q], d[s, q]))
            d[s, q], ids[s, q] = d[s, q, o], ids[s, q, o]
    td, ti, th = (torch.from_numpy(x).cuda() for x in (d, ids, hits))
    od = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    oi = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    oh = torch.empty(nq, dtype=torch.int32, device="cuda")
    gpu.merge_topk_device(td, ti, th, k, od, oi, oh)
    torch.cuda.synchronize()
    wd, wi, wh = merge_reference(d, ids, hits, k)
    assert np.array_equal(oh.cpu().numpy(), wh)
    for q in range(nq):
        m = wh[q]
        assert np.array_equal(oi.cpu().numpy()[q, :m], wi[q, :m])
        assert np.array_equal(od.cpu().numpy()[q, :m], wd[q, :m])
