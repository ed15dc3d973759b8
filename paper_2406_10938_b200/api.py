"""Host-side mirror of the reference's C++ API for the DET-LSH hot path.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/detlsh/{index,projection,encoder,de_tree}.hpp:

    build_index(data, params, seed)                 index.hpp:39
    build_index_with_family(data, params, family, seed)   index.hpp:42-43
    ck_ann(index, q, k) -> QueryResult              index.hpp:87
    candidate_budget(beta, n, k)                    index.hpp:50
    derive_params(K, c, L)                          projection.hpp:75-77
    sample_hash_family(d, K, L, seed)               projection.hpp:30
    project_dataset(family, data)                   projection.hpp:58
    select_breakpoints(projected, n_regions, sample_fraction, seed)  encoder.hpp:41-42
    encode_dataset(projected, table)                encoder.hpp:63
    build_tree(encoded, space, max_size)            de_tree.hpp:61

plus ``ck_ann_batch`` (the batched GPU entry point).  std::invalid_argument
maps to ValueError; device failures to RuntimeError.  Every call goes through
the C ABI (include/detlsh_b200.h) into the sm_100a kernels.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from ._lib import (F_BORROW_DATA, F_DEVICE_PTRS, F_NO_CODES, F_NO_TC, F_NO_U8, F_PAA, F_SAMPLE_GPU,
                   Params, check)

SAMPLE_REFERENCE = "reference"
SAMPLE_GPU = "gpu"


@dataclass
class LshParams:
    """detlsh::LshParams (projection.hpp:79-92)."""

    K: int = 16
    L: int = 4
    c: float = 1.5
    beta: float = 0.0  # <= 0: derived at build
    epsilon: float = 0.0
    alpha1: float = 0.0
    alpha2: float = 0.0
    n_regions: int = 256
    sample_fraction: float = 0.1
    leaf_capacity: int = 128
    r_min: float = 0.0  # <= 0: estimated at build
    k: int = 50

    def to_c(self) -> Params:
        return Params(*[getattr(self, f.name) for f in fields(self)])

    @staticmethod
    def from_c(p: Params) -> "LshParams":
        return LshParams(*[getattr(p, f.name) for f in fields(LshParams)])


@dataclass
class DerivedParams:
    alpha1: float
    alpha2: float
    epsilon: float
    beta: float


@dataclass
class QueryResult:
    """detlsh::QueryResult (index.hpp:79-83)."""

    hits: list = field(default_factory=list)  # [(position, distance)] ascending
    radius_used: float = 0.0
    candidates_seen: int = 0


@dataclass
class TreeExport:
    """A DeTree (de_tree.hpp:44-58) flattened; nodes in the reference's build order."""

    root_children: np.ndarray
    is_leaf: np.ndarray
    split_dim: np.ndarray
    left: np.ndarray
    right: np.ndarray
    bits: np.ndarray
    value: np.ndarray
    ebegin: np.ndarray
    ecount: np.ndarray
    positions: np.ndarray


def _ptr(a) -> C.c_void_p:
    return C.c_void_p(a.ctypes.data)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


def _as_host_f32(x, ndim=2) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    if a.ndim != ndim:
        raise ValueError(f"expected a {ndim}-d array, got shape {a.shape}")
    return a


def _check_tensor(t, name: str, dtype, shape, device: int | None = None):
    """A CUDA tensor the C ABI reads or writes through a raw pointer: its dtype,
    shape and layout must be exactly what the library assumes."""
    import torch
    if not _is_cuda_tensor(t):
        raise ValueError(f"{name}: expected a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name}: expected dtype {dtype}, got {t.dtype}")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    if device is not None and t.device.index != device:
        raise ValueError(f"{name}: tensor is on cuda:{t.device.index}, the index on cuda:{device}")
    del torch


def candidate_budget(beta: float, n: int, k: int) -> int:
    return int(_lib.load().detlsh_candidate_budget(beta, n, k))


def derive_params(K: int, c: float, L: int) -> DerivedParams:
    out = np.empty(4, np.float64)
    check(_lib.load().detlsh_derive_params(K, c, L, _ptr(out)))
    return DerivedParams(*map(float, out))


def chi2_cdf(x: float, k: int) -> float:
    return float(_lib.load().detlsh_chi2_cdf(x, k))


def chi2_quantile(alpha: float, k: int) -> float:
    return float(_lib.load().detlsh_chi2_quantile(alpha, k))


def mix_seed(seed: int, stream: int) -> int:
    """rng.hpp:56-61 (host arithmetic, for callers that derive stage seeds)."""
    m = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15 * (stream + 1)) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def sample_hash_family(d: int, K: int, L: int, seed: int) -> np.ndarray:
    out = np.empty((L, K, d), np.float32)
    check(_lib.load().detlsh_sample_hash_family(d, K, L, seed, _ptr(out)))
    return out


def device_count() -> int:
    return int(_lib.load().detlsh_device_count())


class DetIndex:
    """Assembled GPU index (detlsh::DetIndex, index.hpp:24-37).  Immutable after build."""

    def __init__(self, handle, params: LshParams, n: int, d: int, device: int, owner=None):
        self._h = handle
        self.params = params
        self._n, self._d, self.device = n, d, device
        self._owner = owner  # borrowed handle (a shard of a ShardedIndex): never freed here

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and getattr(self, "_owner", None) is None:
            try:
                _lib.load().detlsh_gpu_free(h)
            except Exception:
                pass
            self._h = None

    def n(self) -> int:
        return self._n

    def d(self) -> int:
        return self._d

    @property
    def handle(self):
        return self._h

    def sample_size(self) -> int:
        return int(_lib.load().detlsh_gpu_sample_size(self._h))

    def row_u8(self) -> int:
        """Bytes per exact-u8 verification row (0: fp64 verification only)."""
        return int(_lib.load().detlsh_gpu_row_u8(self._h))

    def table(self) -> np.ndarray:
        p = self.params
        out = np.empty((p.L, p.K, p.n_regions + 1), np.float32)
        check(_lib.load().detlsh_gpu_export_table(self._h, _ptr(out)))
        return out

    def family(self) -> np.ndarray:
        p = self.params
        out = np.empty((p.L, p.K, self._d), np.float32)
        check(_lib.load().detlsh_gpu_export_family(self._h, _ptr(out)))
        return out

    def codes(self) -> np.ndarray:
        p = self.params
        out = np.empty((p.L, self._n, p.K), np.uint8)
        check(_lib.load().detlsh_gpu_export_codes(self._h, _ptr(out)))
        return out

    def tree(self, i: int) -> TreeExport:
        lib = _lib.load()
        nn = C.c_uint64(0)
        check(lib.detlsh_gpu_tree_num_nodes(self._h, i, C.byref(nn)))
        return _export_tree(lambda *a: lib.detlsh_gpu_export_tree(self._h, i, *a), self.params.K,
                            nn.value, self._n)

    def save_index(self, path: str | None = None) -> bytes:
        """save_index (persist.hpp:17): the DETL v1 bytes the reference writes for
        this index; also written to `path` when given."""
        lib = _lib.load()
        size = C.c_uint64(0)
        check(lib.detlsh_gpu_save_detl(self._h, None, 0, C.byref(size)))
        buf = np.empty(size.value, np.uint8)
        check(lib.detlsh_gpu_save_detl(self._h, _ptr(buf), size.value, C.byref(size)))
        b = buf.tobytes()
        if path is not None:
            with open(path, "wb") as f:
                f.write(b)
        return b

    def build_timings(self) -> dict:
        ms = np.zeros(32, np.float64)
        names = C.create_string_buffer(1024)
        m = _lib.load().detlsh_gpu_build_timings(self._h, _ptr(ms), 32, names, 1024)
        keys = names.value.decode().split(";") if m else []
        return {k: float(v) for k, v in zip(keys, ms[:m])}

    def project_query(self, q, space: int) -> np.ndarray:
        """DetIndex::project_query (index.cpp:181-188) via the projection kernel."""
        return self.project_queries(np.asarray(q, np.float32).reshape(1, -1))[space, 0]

    def project_queries(self, queries) -> np.ndarray:
        """project_query for a batch: [L][nq][K] (detlsh_gpu_project_query)."""
        Q = _as_host_f32(queries)
        if Q.shape[1] != self._d:
            raise ValueError("project_query: query dimension mismatch")
        out = np.empty((self.params.L, Q.shape[0], self.params.K), np.float32)
        check(_lib.load().detlsh_gpu_project_query(self._h, _ptr(Q), Q.shape[0], _ptr(out), 0))
        return out


def _export_tree(fn, K, nn, n) -> TreeExport:
    t = TreeExport(np.empty(1 << K, np.int32), np.empty(nn, np.uint8), np.empty(nn, np.uint8),
                   np.empty(nn, np.int32), np.empty(nn, np.int32), np.empty((nn, K), np.uint8),
                   np.empty((nn, K), np.uint8), np.empty(nn, np.uint64), np.empty(nn, np.uint32),
                   np.empty(n, np.uint32))
    check(fn(_ptr(t.root_children), _ptr(t.is_leaf), _ptr(t.split_dim), _ptr(t.left),
             _ptr(t.right), _ptr(t.bits), _ptr(t.value), _ptr(t.ebegin), _ptr(t.ecount),
             _ptr(t.positions)))
    return t


def _flags(sample: str) -> int:
    if sample not in (SAMPLE_REFERENCE, SAMPLE_GPU):
        raise ValueError(f"sample must be '{SAMPLE_REFERENCE}' or '{SAMPLE_GPU}'")
    return F_SAMPLE_GPU if sample == SAMPLE_GPU else 0


def build_index(data, params: LshParams | None = None, seed: int = 0, *, device: int = 0,
                sample: str = SAMPLE_REFERENCE, borrow: bool = False,
                keep_codes: bool = True, u8_rows: bool = True) -> DetIndex:
    """build_index (index.hpp:39).  `data` is an (n, d) float32 array or a CUDA tensor."""
    params = params or LshParams()
    cp = params.to_c()
    h = C.c_void_p()
    flags = _flags(sample) | (0 if keep_codes else F_NO_CODES) | (0 if u8_rows else F_NO_U8)
    if _is_cuda_tensor(data):
        import torch
        if data.dim() != 2:
            raise ValueError(f"build_index: expected a 2-d tensor, got shape {tuple(data.shape)}")
        if data.dtype != torch.float32:
            raise ValueError(f"build_index: expected float32 points, got {data.dtype}")
        t = data.contiguous()
        n, d = int(t.shape[0]), int(t.shape[1])
        flags |= F_DEVICE_PTRS | (F_BORROW_DATA if borrow else 0)
        dev = t.device.index if t.device.index is not None else device
        check(_lib.load().detlsh_gpu_build(C.c_void_p(t.data_ptr()), n, d, C.byref(cp), seed, dev,
                                           flags, C.byref(h)))
        idx = DetIndex(h, LshParams.from_c(cp), n, d, dev)
        if borrow:
            idx._keepalive = t
        return idx
    a = _as_host_f32(data)
    n, d = a.shape
    check(_lib.load().detlsh_gpu_build(_ptr(a), n, d, C.byref(cp), seed, device, flags,
                                       C.byref(h)))
    return DetIndex(h, LshParams.from_c(cp), n, d, device)


def build_index_with_family(data, params: LshParams, family: np.ndarray, seed: int = 0, *,
                            family_seed: int = 0, device: int = 0,
                            sample: str = SAMPLE_REFERENCE) -> DetIndex:
    """build_index_with_family (index.hpp:42-43): the family's d/K/L win."""
    a = _as_host_f32(data)
    fam = np.ascontiguousarray(family, np.float32)
    L, K, d = fam.shape
    if d != a.shape[1]:
        raise ValueError("build_index: family dimension does not match the dataset")
    cp = params.to_c()
    h = C.c_void_p()
    check(_lib.load().detlsh_gpu_build_with_family(_ptr(a), a.shape[0], d, C.byref(cp), _ptr(fam),
                                                   K, L, family_seed, seed, device,
                                                   _flags(sample), C.byref(h)))
    return DetIndex(h, LshParams.from_c(cp), a.shape[0], d, device)


@dataclass
class BatchResult:
    ids: np.ndarray        # [nq][k] u32
    dists: np.ndarray      # [nq][k] f64
    n_hits: np.ndarray     # [nq] i32
    radius_used: np.ndarray  # [nq] f64
    candidates_seen: np.ndarray  # [nq] u64

    def result(self, i: int) -> QueryResult:
        m = int(self.n_hits[i])
        return QueryResult([(int(p), float(v)) for p, v in zip(self.ids[i, :m], self.dists[i, :m])],
                           float(self.radius_used[i]), int(self.candidates_seen[i]))


def ck_ann_batch(index: DetIndex, queries, k: int, *, stream=None,
                 tensor_cores: bool = True, out: BatchResult | None = None) -> BatchResult:
    """Batched ck_ann over host queries [nq][d] (outputs on the host).

    tensor_cores=False keeps verification on the per-query gather path (no
    tcgen05 dataset-major scoring); the results are identical either way.
    `out`: caller-owned result arrays (e.g. page-locked, reused across
    batches); shapes [nq][k] / [nq], dtypes as in BatchResult."""
    Q = _as_host_f32(queries)
    if Q.shape[1] != index.d():
        raise ValueError("ck_ann: query dimension mismatch")
    nq = Q.shape[0]
    if out is None:
        out = BatchResult(np.zeros((nq, k), np.uint32), np.zeros((nq, k), np.float64),
                          np.zeros(nq, np.int32), np.zeros(nq, np.float64), np.zeros(nq, np.uint64))
    else:
        want = ((out.ids, np.uint32, (nq, k)), (out.dists, np.float64, (nq, k)), (out.n_hits, np.int32, (nq,)),
                (out.radius_used, np.float64, (nq,)), (out.candidates_seen, np.uint64, (nq,)))
        for arr, dt, shape in want:
            if arr.dtype != dt or arr.shape != shape or not arr.flags["C_CONTIGUOUS"]:
                raise ValueError(f"ck_ann: out array must be {np.dtype(dt).name} {shape} C-contiguous")
    flags = 0 if tensor_cores else F_NO_TC
    check(_lib.load().detlsh_gpu_query(index.handle, _ptr(Q), nq, k, flags, _ptr(out.ids),
                                       _ptr(out.dists), _ptr(out.n_hits), _ptr(out.radius_used),
                                       _ptr(out.candidates_seen), stream))
    return out


def ck_ann_device(index: DetIndex, queries, k: int, ids, dists, n_hits=None, radius=None,
                  cands=None, stream=None, tensor_cores: bool = True) -> None:
    """Batched ck_ann on device tensors (stream-ordered, no host copies)."""
    import torch

    def p(t):
        return C.c_void_p(t.data_ptr()) if t is not None else None
    if queries.dim() != 2 or queries.shape[1] != index.d():
        raise ValueError("ck_ann: query dimension mismatch")
    nq = int(queries.shape[0])
    dev = index.device
    _check_tensor(queries, "ck_ann: queries", torch.float32, (nq, index.d()), dev)
    _check_tensor(ids, "ck_ann: ids", torch.int32, (nq, k), dev)
    _check_tensor(dists, "ck_ann: dists", torch.float64, (nq, k), dev)
    for t, name, dt in ((n_hits, "n_hits", torch.int32), (radius, "radius", torch.float64),
                        (cands, "cands", torch.int64)):
        if t is not None:
            _check_tensor(t, f"ck_ann: {name}", dt, (nq,), dev)
    flags = F_DEVICE_PTRS | (0 if tensor_cores else F_NO_TC)
    check(_lib.load().detlsh_gpu_query(index.handle, p(queries), nq, k, flags, p(ids), p(dists),
                                       p(n_hits), p(radius), p(cands), stream))


def query_check(index: DetIndex, stream=None) -> None:
    """Synchronise and raise if an earlier device-pointer batch failed an internal check."""
    check(_lib.load().detlsh_gpu_query_check(index.handle, stream))


def estimate_rmin(index: DetIndex, probes, k: int) -> float:
    """estimate_rmin (index.hpp:91, index.cpp:333-374) over probe queries [np][d]."""
    P = _as_host_f32(probes)
    if P.shape[0] and P.shape[1] != index.d():
        raise ValueError("estimate_rmin: probe dimension mismatch")
    out = C.c_double(0.0)
    check(_lib.load().detlsh_gpu_estimate_rmin(index.handle, _ptr(P), P.shape[0], k, 0, C.byref(out)))
    return float(out.value)


def _range_query(index: DetIndex, tree: int, q_proj, radius, limit: int, exact: bool, cap=None):
    qp = np.ascontiguousarray(np.atleast_2d(np.asarray(q_proj, np.float32)))
    nq = qp.shape[0]
    if qp.shape[1] != index.params.K:
        raise ValueError("range_query: projected query must have K coordinates")
    rad = np.ascontiguousarray(np.broadcast_to(np.asarray(radius, np.float64), (nq,)))
    cap = min(index.n(), limit) if cap is None else cap
    out = np.zeros((nq, max(1, cap)), np.uint32)
    counts = np.zeros(nq, np.uint64)
    check(_lib.load().detlsh_gpu_range_query(index.handle, tree, _ptr(qp), nq, _ptr(rad), limit,
                                             _lib.RANGE_EXACT if exact else 0, _ptr(out), cap, _ptr(counts)))
    return [out[i, :min(int(counts[i]), cap)].copy() for i in range(nq)]


def range_query_optimized(index: DetIndex, tree: int, q_proj, radius: float, limit: int = 2**63):
    """range_query_optimized (de_tree.hpp:93-100) with a sink that stops after
    `limit` positions: the entries of every leaf with mindist <= radius in
    ascending (mindist, node index) order."""
    return _range_query(index, tree, q_proj, radius, limit, False)[0]


def range_query_exact(index: DetIndex, tree: int, q_proj, radius: float):
    """range_query_exact (de_tree.hpp:85-91): {pos : ||q', o'_pos|| <= radius} in DFS order."""
    return _range_query(index, tree, q_proj, radius, 2**63, True)[0]


def brute_force_knn(data, queries, k: int, *, dist2_bound=None, device: int = 0):
    """brute_force_knn (metrics.cpp:8-33) on the GPU: (ids [nq][k], dists [nq][k])
    ordered by (dist^2, position).  dist2_bound: optional per-query upper bound
    on the k-th smallest dist^2 (e.g. the squared k-th ck_ann distance)."""
    X = _as_host_f32(data)
    Q = _as_host_f32(queries)
    if Q.shape[1] != X.shape[1]:
        raise ValueError("brute_force_knn: query dimension mismatch")
    nq = Q.shape[0]
    ids = np.zeros((nq, k), np.uint32)
    ds = np.zeros((nq, k), np.float64)
    b = None
    if dist2_bound is not None:
        bound = np.ascontiguousarray(dist2_bound, np.float64)
        b = _ptr(bound)
    check(_lib.load().detlsh_gpu_brute_force_knn(_ptr(X), X.shape[0], X.shape[1], _ptr(Q), nq, k, b, 0,
                                                 _ptr(ids), _ptr(ds), device, None))
    return ids, ds


def brute_force_knn_device(data, queries, k: int, *, dist2_bound=None, stream=None):
    """brute_force_knn on CUDA tensors (data [n][d], queries [nq][d] fp32 on one
    device): (ids [nq][k] uint32 as int32 tensor, dists [nq][k] float64 tensor)."""
    import torch
    dev = data.device.index if data.device.index is not None else 0
    n, d = data.shape
    nq = int(queries.shape[0])
    _check_tensor(data, "brute_force_knn: data", torch.float32, (n, d), dev)
    _check_tensor(queries, "brute_force_knn: queries", torch.float32, (nq, d), dev)
    ids = torch.empty((nq, k), dtype=torch.int32, device=data.device)
    ds = torch.empty((nq, k), dtype=torch.float64, device=data.device)
    b = None
    if dist2_bound is not None:
        bt = torch.as_tensor(dist2_bound, dtype=torch.float64, device=data.device).contiguous()
        b = C.c_void_p(bt.data_ptr())
    check(_lib.load().detlsh_gpu_brute_force_knn(C.c_void_p(data.data_ptr()), n, d, C.c_void_p(queries.data_ptr()),
                                                 nq, k, b, F_DEVICE_PTRS, C.c_void_p(ids.data_ptr()),
                                                 C.c_void_p(ds.data_ptr()), dev, stream))
    return ids, ds


def vectors_shape(path: str):
    """(n, d, kind) of a .fvecs / .bvecs / .ivecs file (io.cpp:28-85 validation)."""
    n = C.c_uint64(0)
    d = C.c_int32(0)
    kind = C.c_int32(0)
    check(_lib.load().detlsh_vectors_shape(path.encode(), C.byref(n), C.byref(d), C.byref(kind)))
    return n.value, d.value, ("f32", "u8", "i32")[kind.value]


def read_vectors_device(path: str, device: int = 0):
    """read_vectors (io.hpp) straight into a CUDA tensor [n][d] fp32: the file
    streams through pinned chunks, u8 / i32 elements are widened on the GPU."""
    import torch
    n, d, _ = vectors_shape(path)
    out = torch.empty((n, d), dtype=torch.float32, device=f"cuda:{device}")
    if n:
        check(_lib.load().detlsh_gpu_read_vectors(path.encode(), C.c_void_p(out.data_ptr()), n, d, device,
                                                  None))
    return out


def rc_ann_batch(index: DetIndex, queries, r: float, c: float):
    """rc_ann (index.cpp:267-290) for a batch of host queries [nq][d]: returns
    (ids [nq] u32, dists [nq] f64, found [nq] bool, candidates_seen [nq])."""
    Q = _as_host_f32(queries)
    if Q.shape[1] != index.d():
        raise ValueError("rc_ann: query dimension mismatch")
    nq = Q.shape[0]
    ids = np.zeros(nq, np.uint32)
    ds = np.zeros(nq, np.float64)
    found = np.zeros(nq, np.int32)
    cs = np.zeros(nq, np.uint64)
    check(_lib.load().detlsh_gpu_rc_ann(index.handle, _ptr(Q), nq, float(r), float(c), 0, _ptr(ids),
                                        _ptr(ds), _ptr(found), _ptr(cs), None))
    return ids, ds, found.astype(bool), cs


def rc_ann(index: DetIndex, q, r: float, c: float):
    """rc_ann (index.hpp, index.cpp:267-290): (position, distance) or None."""
    ids, ds, found, _ = rc_ann_batch(index, np.asarray(q, np.float32).reshape(1, -1), r, c)
    return (int(ids[0]), float(ds[0])) if found[0] else None


def build_det_only_index(data, params: LshParams | None = None, seed: int = 0, *, device: int = 0,
                         sample: str = SAMPLE_REFERENCE) -> DetIndex:
    """build_det_only_index (index.cpp:220-232): the DET-ONLY variant -- PAA
    segment means (projection.cpp:62-90) as the single projected space (L = 1)."""
    params = params or LshParams()
    cp = params.to_c()
    a = _as_host_f32(data)
    h = C.c_void_p()
    check(_lib.load().detlsh_gpu_build(_ptr(a), a.shape[0], a.shape[1], C.byref(cp), seed, device,
                                       _flags(sample) | F_PAA, C.byref(h)))
    return DetIndex(h, LshParams.from_c(cp), a.shape[0], a.shape[1], device)


def ck_ann(index: DetIndex, q, k: int) -> QueryResult:
    """ck_ann (index.hpp:87, index.cpp:292-331) for one query."""
    qa = np.asarray(q, np.float32).reshape(1, -1)
    if qa.shape[1] != index.d():
        raise ValueError("ck_ann: query dimension mismatch")
    return ck_ann_batch(index, qa, k).result(0)


def merge_topk_device(shard_dists, shard_ids, shard_hits, k: int, out_dists, out_ids, out_hits,
                      stream=None) -> None:
    """Merge per-shard top-k lists ([shards][nq][k], device tensors) into the global top-k."""
    import torch
    shards, nq = int(shard_dists.shape[0]), int(shard_dists.shape[1])
    _check_tensor(shard_dists, "merge_topk: shard_dists", torch.float64, (shards, nq, k))
    _check_tensor(shard_ids, "merge_topk: shard_ids", torch.int64, (shards, nq, k))
    _check_tensor(shard_hits, "merge_topk: shard_hits", torch.int32, (shards, nq))
    _check_tensor(out_dists, "merge_topk: out_dists", torch.float64, (nq, k))
    _check_tensor(out_ids, "merge_topk: out_ids", torch.int64, (nq, k))
    _check_tensor(out_hits, "merge_topk: out_hits", torch.int32, (nq,))
    check(_lib.load().detlsh_gpu_merge_topk(
        C.c_void_p(shard_dists.data_ptr()), C.c_void_p(shard_ids.data_ptr()),
        C.c_void_p(shard_hits.data_ptr()), shards, nq, k, C.c_void_p(out_dists.data_ptr()),
        C.c_void_p(out_ids.data_ptr()), C.c_void_p(out_hits.data_ptr()), stream))


class ShardedIndex:
    """Point-sharded index in one process (detlsh_gpu_sharded_*):
    shard s = rows [s*n/S, (s+1)*n/S) on devices[s], an independent DET-LSH
    index; queries merge per (distance, global position) on devices[0]."""

    def __init__(self, handle, params: LshParams, n: int, d: int, devices):
        self._h = handle
        self.params = params
        self.n, self.d, self.devices = n, d, list(devices)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.load().detlsh_gpu_sharded_free(h)
            except Exception:
                pass
            self._h = None

    def shard(self, s: int) -> DetIndex:
        """Borrowed view of shard s (a DetIndex: export, per-shard queries)."""
        lib = _lib.load()
        b, e = C.c_uint64(0), C.c_uint64(0)
        h = lib.detlsh_gpu_sharded_shard(self._h, s, C.byref(b), C.byref(e))
        if not h:
            raise ValueError("no such shard")
        cp = Params()
        check(lib.detlsh_gpu_get_params(h, C.byref(cp)))
        v = DetIndex(C.c_void_p(h), LshParams.from_c(cp), e.value - b.value, self.d, self.devices[s], owner=self)
        v.rows = (b.value, e.value)
        return v

    def shard_count(self) -> int:
        return int(_lib.load().detlsh_gpu_sharded_count(self._h))


def build_sharded_index(data, params: LshParams | None = None, seed: int = 0, *, devices=(0,),
                        sample: str = SAMPLE_REFERENCE) -> ShardedIndex:
    """build_index per contiguous point shard, concurrently on `devices`
    (one shard per entry; a device may appear several times)."""
    params = params or LshParams()
    cp = params.to_c()
    a = _as_host_f32(data)
    devs = np.ascontiguousarray(devices, np.int32)
    h = C.c_void_p()
    check(_lib.load().detlsh_gpu_sharded_build(_ptr(a), a.shape[0], a.shape[1], C.byref(cp), seed,
                                               _ptr(devs), len(devs), _flags(sample), C.byref(h)))
    return ShardedIndex(h, LshParams.from_c(cp), a.shape[0], a.shape[1], devs.tolist())


def ck_ann_sharded(index: ShardedIndex, queries, k: int, *, tensor_cores: bool = True):
    """Batched ck_ann over every shard + merge: (ids [nq][k] u64 global positions,
    dists [nq][k] f64, n_hits [nq] i32), ascending by (distance, position)."""
    Q = _as_host_f32(queries)
    if Q.shape[1] != index.d:
        raise ValueError("ck_ann: query dimension mismatch")
    nq = Q.shape[0]
    ids = np.zeros((nq, k), np.uint64)
    ds = np.zeros((nq, k), np.float64)
    nh = np.zeros(nq, np.int32)
    check(_lib.load().detlsh_gpu_sharded_query(index._h, _ptr(Q), nq, k, 0 if tensor_cores else F_NO_TC,
                                               _ptr(ids), _ptr(ds), _ptr(nh), None))
    return ids, ds, nh


def ck_ann_sharded_device(index: ShardedIndex, queries, k: int, ids, dists, n_hits, stream=None) -> None:
    """Stream-ordered sharded ck_ann on CUDA tensors of devices[0]."""
    import torch
    nq = int(queries.shape[0])
    dev = index.devices[0]
    _check_tensor(queries, "ck_ann: queries", torch.float32, (nq, index.d), dev)
    _check_tensor(ids, "ck_ann: ids", torch.int64, (nq, k), dev)
    _check_tensor(dists, "ck_ann: dists", torch.float64, (nq, k), dev)
    _check_tensor(n_hits, "ck_ann: n_hits", torch.int32, (nq,), dev)
    check(_lib.load().detlsh_gpu_sharded_query(index._h, C.c_void_p(queries.data_ptr()), nq, k, F_DEVICE_PTRS,
                                               C.c_void_p(ids.data_ptr()), C.c_void_p(dists.data_ptr()),
                                               C.c_void_p(n_hits.data_ptr()), stream))


# ---- stage functions ----------------------------------------------------------------

def project_dataset(family: np.ndarray, data, *, device: int = 0) -> np.ndarray:
    """project_dataset (projection.hpp:58) -> [L][n][K] fp32, bit-exact."""
    fam = np.ascontiguousarray(family, np.float32)
    L, K, d = fam.shape
    a = _as_host_f32(data)
    if a.shape[1] != d:
        raise ValueError("project_dataset: dataset dimension mismatch")
    out = np.empty((L, a.shape[0], K), np.float32)
    check(_lib.load().detlsh_gpu_project(_ptr(fam), K, L, _ptr(a), a.shape[0], d, _ptr(out),
                                         device, 0))
    return out


def select_breakpoints(projected: np.ndarray, n_regions: int, sample_fraction: float, seed: int,
                       *, device: int = 0, sample: str = SAMPLE_REFERENCE) -> np.ndarray:
    """select_breakpoints (encoder.hpp:41-42) -> [L][K][n_regions+1]."""
    pr = np.ascontiguousarray(projected, np.float32)
    L, n, K = pr.shape
    out = np.empty((L, K, n_regions + 1), np.float32)
    ns = C.c_uint64(0)
    check(_lib.load().detlsh_gpu_select_breakpoints(_ptr(pr), n, K, L, n_regions, sample_fraction,
                                                    seed, _ptr(out), C.byref(ns), device,
                                                    _flags(sample)))
    return out


def encode_dataset(projected: np.ndarray, table: np.ndarray, *, device: int = 0) -> np.ndarray:
    """encode_dataset (encoder.hpp:63) -> [L][n][K] u8."""
    pr = np.ascontiguousarray(projected, np.float32)
    tb = np.ascontiguousarray(table, np.float32)
    L, n, K = pr.shape
    if tb.shape[:2] != (L, K):
        raise ValueError("encode_dataset: table shape does not match projected dataset")
    out = np.empty((L, n, K), np.uint8)
    check(_lib.load().detlsh_gpu_encode(_ptr(pr), n, K, L, _ptr(tb), tb.shape[2] - 1, _ptr(out),
                                        device, 0))
    return out


def build_tree(encoded: np.ndarray, space: int, max_size: int, n_regions: int = 256, *,
               device: int = 0) -> TreeExport:
    """build_tree (de_tree.hpp:61) on the GPU, exported in the reference layout."""
    enc = np.ascontiguousarray(encoded, np.uint8)
    L, n, K = enc.shape
    lib = _lib.load()
    h = C.c_void_p()
    check(lib.detlsh_gpu_build_tree(_ptr(enc), n, K, L, n_regions, space, max_size, device, 0,
                                    C.byref(h)))
    try:
        nn = C.c_uint64(0)
        check(lib.detlsh_gpu_tree_nodes(h, C.byref(nn)))
        return _export_tree(lambda *a: lib.detlsh_gpu_tree_export(h, *a), K, nn.value, n)
    finally:
        lib.detlsh_gpu_tree_free(h)
