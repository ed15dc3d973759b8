"""Point sharding across ranks: contiguous row ranges, one
independent DET-LSH index per rank, queries broadcast, per-shard top-k lists
exchanged with one all-gather and merged by (distance, global id) on the GPU
(detlsh_gpu_merge_topk).  torch.distributed is the plumbing (NCCL on the GPU
box; gloo in the CPU tests)."""
from __future__ import annotations


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    return rank * n // world, (rank + 1) * n // world


def gather_topk(dists, gids, hits, out_d, out_i, out_h, group=None) -> None:
    """All-gather per-shard top-k lists: [nq][k] -> [world][nq][k] (rank order)."""
    import torch.distributed as dist
    for src, dst in ((dists, out_d), (gids, out_i), (hits, out_h)):
        dist.all_gather_into_tensor(dst.view(-1, *src.shape[1:]), src, group=group)
