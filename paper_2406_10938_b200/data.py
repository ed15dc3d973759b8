"""Seeded synthetic stand-ins for BASELINE.json's configs (none of the paper's
datasets are in this environment).  Each generator returns (base, queries) as
float32 arrays; queries are held out from the same distribution (the last nq
rows of one draw).  numpy PCG64 streams make every byte reproducible.

  C1  n=1e5, d=128: 100 centres U[0,100]^d, isotropic sigma=5, seed 1
  C2  n=1e6, d=128: 0 w.p. 0.5 else min(255, geometric(p=0.05)), seed 2
  C3  n=1e6, d=784: 28x28 grid, 3-6 blobs of radius 3-6, non-zeros U[1,255], seed 3
  C4  n=1e7, d=96 : N(0,1) rows L2-normalised, seed 4
  C5  n=1e8, d=128: the C2 distribution, seed 5, generated on the GPU
      (make_device: a counter-based hash per element, csrc/synth.cu; the
      51 GB dataset never passes through host memory)
"""
from __future__ import annotations

import numpy as np

CONFIGS = {
    "c1": dict(n=100_000, d=128, nq=1_000, seed=1),
    "c2": dict(n=1_000_000, d=128, nq=10_000, seed=2),
    "c3": dict(n=1_000_000, d=784, nq=10_000, seed=3),
    "c4": dict(n=10_000_000, d=96, nq=10_000, seed=4),
    "c5": dict(n=100_000_000, d=128, nq=10_000, seed=5),
}


def mixture(total: int, d: int, seed: int, clusters: int = 100, lo: float = 0.0,
            hi: float = 100.0, sigma: float = 5.0, sample_seed: int | None = None) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    centres = rng.uniform(lo, hi, size=(clusters, d)).astype(np.float32)
    if sample_seed is not None:  # same centres, another draw of members
        rng = np.random.Generator(np.random.PCG64(sample_seed))
    pick = rng.integers(0, clusters, size=total)
    out = np.empty((total, d), np.float32)
    step = 1 << 16
    for s in range(0, total, step):
        e = min(total, s + step)
        out[s:e] = centres[pick[s:e]] + rng.normal(0.0, sigma, size=(e - s, d)).astype(np.float32)
    return out


def sparse_geometric(total: int, d: int, seed: int, p: float = 0.05) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((total, d), np.float32)
    step = 1 << 16
    for s in range(0, total, step):
        e = min(total, s + step)
        zero = rng.random((e - s, d)) < 0.5
        g = np.minimum(rng.geometric(p, size=(e - s, d)), 255)
        out[s:e] = np.where(zero, 0, g).astype(np.float32)
    return out


def blobs784(total: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    g28 = np.arange(28, dtype=np.float32)
    out = np.zeros((total, 784), np.float32)
    step = 1 << 13
    for s in range(0, total, step):
        e = min(total, s + step)
        m = e - s
        nb = rng.integers(3, 7, size=m)
        mask = np.zeros((m, 28, 28), bool)
        for b in range(6):
            active = nb > b
            ctr = rng.uniform(0, 27, size=(m, 2)).astype(np.float32)
            rad = rng.uniform(3, 6, size=m).astype(np.float32)
            # squared distance of grid cell (y, x) to the blob centre, in float32
            dy2 = (g28[None, :] - ctr[:, 0:1]) ** 2
            dx2 = (g28[None, :] - ctr[:, 1:2]) ** 2
            d2 = dy2[:, :, None] + dx2[:, None, :]
            mask |= active[:, None, None] & (d2 < 0.5 * (rad ** 2)[:, None, None])
        vals = rng.integers(1, 256, size=(m, 784)).astype(np.float32)
        out[s:e] = np.where(mask.reshape(m, 784), vals, 0.0)
    return out


def unit_gaussian(total: int, d: int, seed: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    out = np.empty((total, d), np.float32)
    step = 1 << 18
    for s in range(0, total, step):
        e = min(total, s + step)
        x = rng.standard_normal((e - s, d), dtype=np.float32)
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        out[s:e] = x
    return out


def make(config: str, n: int | None = None, nq: int | None = None):
    """(base [n][d], queries [nq][d]) for config c1..c5 (n/nq may be scaled down)."""
    c = CONFIGS[config]
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    total = n + nq
    if config == "c1":
        allp = mixture(total, c["d"], c["seed"])
    elif config in ("c2", "c5"):
        allp = sparse_geometric(total, c["d"], c["seed"])
    elif config == "c3":
        allp = blobs784(total, c["seed"])
    elif config == "c4":
        allp = unit_gaussian(total, c["d"], c["seed"])
    else:
        raise ValueError(config)
    return allp[:n], allp[n:]


def make_shard(config: str, rank: int, n: int | None = None) -> np.ndarray:
    """Rank `rank`'s n points of the weak-scaling dataset (world x n points): shard 0
    is make(config)'s base, shard r > 0 is an independent draw of the same
    distribution (seed + 1000 r).  The held-out queries stay make(config)'s."""
    c = CONFIGS[config]
    n = c["n"] if n is None else n
    if rank == 0:
        return make(config, n=n)[0]
    seed = c["seed"] + 1000 * rank
    if config == "c1":
        return mixture(n, c["d"], c["seed"], sample_seed=seed)
    if config in ("c2", "c5"):
        return sparse_geometric(n, c["d"], seed)
    if config == "c3":
        return blobs784(n, seed)
    if config == "c4":
        return unit_gaussian(n, c["d"], seed)
    raise ValueError(config)



def make_device(config: str, n: int | None = None, nq: int | None = None, device: int = 0):
    """(base [n][d], queries [nq][d]) as CUDA tensors, generated on the GPU
    (detlsh_gpu_synth kind 0): config c5 (and c2-shaped variants).  Rows
    [0, n) are the base set, rows [n, n + nq) the held-out queries."""
    import ctypes as C

    import torch

    from . import _lib
    c = CONFIGS[config]
    if config not in ("c2", "c5"):
        raise ValueError("device generation covers the sparse 8-bit configs (c2, c5)")
    n = c["n"] if n is None else n
    nq = c["nq"] if nq is None else nq
    d = c["d"]
    base = torch.empty((n, d), dtype=torch.float32, device=f"cuda:{device}")
    Q = torch.empty((nq, d), dtype=torch.float32, device=f"cuda:{device}")
    lib = _lib.load()
    _lib.check(lib.detlsh_gpu_synth(0, c["seed"], 0, n, d, C.c_void_p(base.data_ptr()), device, None))
    _lib.check(lib.detlsh_gpu_synth(0, c["seed"], n, nq, d, C.c_void_p(Q.data_ptr()), device, None))
    return base, Q
