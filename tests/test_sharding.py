"""Multi-rank path on CPU: world_size 2 over gloo.  Each rank builds an
independent index on its contiguous shard (the CPU oracle stands in for the
per-shard GPU index, which is parity-tested separately), answers every query,
offsets ids to global positions, all-gathers the top-k lists and merges them.
The merged answer must equal the merge computed in a single process from the
same per-shard oracle runs (SURVEY §8e parity definition)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import gaussian
from oracle.bindings import Oracle, make_params
from paper_2406_10938_b200.shard import gather_topk, shard_bounds

N, D, NQ, K = 3001, 16, 12, 10
PKW = dict(K=8, L=2, n_regions=16, leaf_capacity=16, sample_fraction=0.5, beta=0.1, k=K)


def merge_reference(dists, ids, hits, k):
    """Ascending (dist, global id) over all shards' lists (the GPU merge's contract)."""
    S, nq, _ = dists.shape
    od = np.zeros((nq, k))
    oi = np.zeros((nq, k), np.int64)
    oh = np.zeros(nq, np.int32)
    for q in range(nq):
        cand = [(dists[s, q, j], ids[s, q, j]) for s in range(S) for j in range(hits[s, q])]
        cand.sort()
        m = min(k, len(cand))
        oh[q] = m
        for j in range(m):
            od[q, j], oi[q, j] = cand[j]
    return od, oi, oh


def shard_topk(rank, world, base, Q):
    s0, s1 = shard_bounds(N, world, rank)
    idx = Oracle("port").build_index(base[s0:s1], make_params(**PKW), 5)
    d = np.zeros((NQ, K))
    i = np.zeros((NQ, K), np.int64)
    h = np.zeros(NQ, np.int32)
    for q in range(NQ):
        ids, ds, _, _ = idx.ck_ann(Q[q], K)
        d[q, :len(ids)], i[q, :len(ids)], h[q] = ds, ids.astype(np.int64) + s0, len(ids)
    return d, i, h


def worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    base, Q = gaussian(N, D, 1, 1.5), gaussian(NQ, D, 2, 1.5)
    d, i, h = shard_topk(rank, world, base, Q)
    gd = torch.zeros((world, NQ, K), dtype=torch.float64)
    gi = torch.zeros((world, NQ, K), dtype=torch.int64)
    gh = torch.zeros((world, NQ), dtype=torch.int32)
    gather_topk(torch.from_numpy(d), torch.from_numpy(i), torch.from_numpy(h), gd, gi, gh)
    if rank == 0:
        od, oi, oh = merge_reference(gd.numpy(), gi.numpy(), gh.numpy(), K)
        np.savez(out, d=od, i=oi, h=oh)
    dist.barrier()
    dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_bounds_cover_exactly():
    for n in (1, 7, 1000, 10**8):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(w - 1))


@pytest.mark.parametrize("world", [2])
def test_two_rank_gloo_gather_and_merge(tmp_path, world):
    out = str(tmp_path / "merged.npz")
    mp.spawn(worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    base, Q = gaussian(N, D, 1, 1.5), gaussian(NQ, D, 2, 1.5)
    parts = [shard_topk(r, world, base, Q) for r in range(world)]
    want = merge_reference(np.stack([p[0] for p in parts]), np.stack([p[1] for p in parts]),
                           np.stack([p[2] for p in parts]), K)
    assert np.array_equal(got["i"], want[1]) and np.array_equal(got["d"], want[0])
    # sharded recall stays close to the single-index answer on this easy set
    full = Oracle("port").build_index(base, make_params(**PKW), 5)
    same = np.mean([len(set(full.ck_ann(Q[q], K)[0].tolist()) & set(got["i"][q].tolist())) / K
                    for q in range(NQ)])
    assert same >= 0.7


def test_weak_scaling_shards():
    """bench.py --shard weak: shard 0 is the N = 1 dataset, shard r > 0 an
    independent draw of the same distribution (the mixture keeps its centres)."""
    from paper_2406_10938_b200 import data as gen
    base = gen.make("c1", n=2000)[0]  # (default nq, as bench.py generates it)
    s0 = gen.make_shard("c1", 0, 2000)
    s1 = gen.make_shard("c1", 1, 2000)
    assert np.array_equal(base, s0)
    assert s1.shape == s0.shape and not np.array_equal(s0, s1)
    # same centres: every shard-1 point lies near one of the 100 centres shard 0 uses
    c = np.random.Generator(np.random.PCG64(gen.CONFIGS["c1"]["seed"])).uniform(0, 100, size=(100, 128))
    d0 = ((s1[:50, None, :] - c[None, :, :].astype(np.float32)) ** 2).sum(-1).min(1)
    assert np.all(d0 < (5.0 * 4) ** 2 * 128)
    g1 = gen.make_shard("c2", 1, 1000)
    assert g1.shape == (1000, 128) and g1.min() >= 0 and g1.max() <= 255


def test_bench_gpus_2_launches_two_ranks():
    """`bench.py --gpus 2` without a torchrun environment re-launches itself
    under torch.distributed.run with two ranks (gloo here), splits the config's
    n into two contiguous point shards (strong scaling by default) and
    all-gathers the per-shard lists; rank 0 reports n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plumbing"],
                         check=True, capture_output=True, text=True, env=env, timeout=240).stdout
    line = json.loads([x for x in out.splitlines() if x.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["shards"] == [[0, 500000], [500000, 1000000]]
    assert line["gathered_ids"] == [0, 500000]
