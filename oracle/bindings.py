"""TEST INFRASTRUCTURE ONLY — ctypes bindings for the CPU oracle.

Two libraries, same surface:
  * ``Oracle(kind="port")``      -> oracle/liboracle.so (C restatement, detlsh_oracle.c)
  * ``Oracle(kind="reference")`` -> oracle/_ref/libdetlsh_ref.so (the unmodified
    reference sources + oracle/ref_shim.cpp, built by ``make -C oracle ref``)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdetlsh_ref.so")
REF_ROOT = "/root/reference/proj"


class Params(C.Structure):
    # Same field order as detlsh::LshParams (projection.hpp:79-92).
    _fields_ = [
        ("K", C.c_int32), ("L", C.c_int32), ("c", C.c_double), ("beta", C.c_double),
        ("epsilon", C.c_double), ("alpha1", C.c_double), ("alpha2", C.c_double),
        ("n_regions", C.c_int32), ("sample_fraction", C.c_double),
        ("leaf_capacity", C.c_int32), ("r_min", C.c_double), ("k", C.c_int32),
    ]


def make_params(K=16, L=4, c=1.5, beta=0.0, n_regions=256, sample_fraction=0.1,
                leaf_capacity=128, r_min=0.0, k=50) -> Params:
    return Params(K, L, c, beta, 0.0, 0.0, 0.0, n_regions, sample_fraction, leaf_capacity,
                  r_min, k)


def build(ref: bool = False) -> None:
    """Build liboracle.so (and the reference .so when the sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    if ref and os.path.isdir(REF_ROOT):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


@dataclass
class TreeExport:
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


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        path = PORT_SO if kind == "port" else REF_SO
        if not os.path.exists(path):
            build(ref=(kind != "port"))
        self.lib = C.CDLL(path)
        self.pre = "orc_" if kind == "port" else "ref_"
        self._sig()

    def f(self, name):
        return getattr(self.lib, self.pre + name)

    def _sig(self):
        vp, u64, i32, dbl = C.c_void_p, C.c_uint64, C.c_int, C.c_double
        sigs = {
            "mix_seed": ([u64, u64], u64),
            "rng_stream": ([u64, u64, vp, vp], None),
            "chi2_cdf": ([dbl, i32], dbl),
            "chi2_quantile": ([dbl, i32], dbl),
            "regularized_gamma_p": ([dbl, dbl], dbl),
            "derive_params": ([i32, dbl, i32, vp], i32),
            "candidate_budget": ([dbl, u64, i32], u64),
            "sample_hash_family": ([i32, i32, i32, u64, vp], None),
            "project_dataset": ([vp, i32, i32, vp, u64, i32, vp], None),
            "select_breakpoints": None,
            "locate_region": ([C.c_float, vp, i32], i32),
            "encode_dataset": ([vp, u64, i32, i32, vp, i32, vp], None),
            "build_tree": ([vp, u64, i32, i32, i32, i32, i32], vp),
            "tree_free": ([vp], None),
            "tree_num_nodes": ([vp], u64),
            "tree_export": ([vp] + [vp] * 10, None),
            "range_query_optimized": None,
            "mindist": None,
            "build_index": None,
            "build_index_with_table": None,
            "index_free": ([vp], None),
            "index_params": ([vp, vp], None),
            "index_table": ([vp, vp], None),
            "ck_ann": ([vp, vp, i32, vp, vp, vp, vp, vp], i32),
            "brute_force_knn": ([vp, u64, i32, vp, u64, i32, vp, vp], None),
        }
        for name, s in sigs.items():
            fn = self.f(name)
            if s is not None:
                fn.argtypes, fn.restype = s
        # handles are pointers: the default int restype would truncate them
        self.f("build_index").restype = vp
        self.f("build_index_with_table").restype = vp
        if self.kind == "port":
            self.f("select_breakpoints").argtypes = [vp, u64, i32, i32, i32, dbl, u64, vp, vp, vp, vp]
            self.f("range_query_optimized").argtypes = [vp, vp, vp, dbl, u64, vp]
            self.f("mindist").argtypes = [vp, i32, vp, vp]
            self.f("build_index").argtypes = [vp, u64, i32, vp, u64]
            self.f("build_index_with_table").argtypes = [vp, u64, i32, vp, u64, vp]
            self.f("select_row_breakpoints").argtypes = [vp, u64, i32, vp, vp]
            self.lib.orc_rng_seed.argtypes = [vp, u64]
        else:
            self.f("select_breakpoints").argtypes = [vp, u64, i32, i32, i32, dbl, u64, vp, vp]
            self.f("range_query_optimized").argtypes = [vp, vp, i32, vp, dbl, u64, vp]
            self.f("mindist").argtypes = [vp, i32, vp, i32, vp]
            self.f("build_index").argtypes = [vp, u64, i32, vp, u64, vp]
            self.f("build_index_with_table").argtypes = [vp, u64, i32, vp, u64, vp, u64]
            self.f("ck_ann_batch").argtypes = [vp, vp, u64, i32, i32, vp, vp, vp, vp, vp, vp]
            self.f("ck_ann_batch").restype = i32
            self.f("index_tree_nodes").argtypes = [vp, i32]
            self.f("index_tree_nodes").restype = u64
            self.f("index_tree_export").argtypes = [vp, i32] + [vp] * 10
            self.f("index_family").argtypes = [vp, vp]
            self.f("index_sample_size").argtypes = [vp]
            self.f("index_sample_size").restype = u64
            self.f("select_row_breakpoints").argtypes = [vp, u64, i32, u64, vp]
            self.f("index_save").argtypes = [vp, vp, u64]
            self.f("index_save").restype = u64
            self.f("index_fingerprint").argtypes = [vp]
            self.f("index_fingerprint").restype = u64
            self.f("index_load").argtypes = [vp, u64, vp, u64, i32]
            self.f("index_load").restype = vp
            self.f("build_det_only_index").argtypes = [vp, u64, i32, vp, u64]
            self.f("build_det_only_index").restype = vp
            self.f("rc_ann").argtypes = [vp, vp, dbl, dbl, vp, vp]
            self.f("rc_ann").restype = i32
            self.f("index_estimate_rmin").argtypes = [vp, vp, u64, i32]
            self.f("index_estimate_rmin").restype = dbl
            self.f("index_project_query").argtypes = [vp, vp, i32, vp]
            self.f("index_project_query").restype = None
            self.f("index_range_query").argtypes = [vp, i32, vp, dbl, u64, i32, vp, u64]
            self.f("index_range_query").restype = u64

    # ---- scalar helpers ------------------------------------------------------
    def mix_seed(self, seed, stream):
        return int(self.f("mix_seed")(seed, stream))

    def rng_stream(self, seed, count):
        u = np.empty(count, np.uint64)
        g = np.empty(count, np.float64)
        self.f("rng_stream")(seed, count, _p(u), _p(g))
        return u, g

    def derive_params(self, K, c, L):
        out = np.empty(4, np.float64)
        assert self.f("derive_params")(K, c, L, _p(out)) == 0
        return dict(alpha1=out[0], alpha2=out[1], epsilon=out[2], beta=out[3])

    def candidate_budget(self, beta, n, k):
        return int(self.f("candidate_budget")(beta, n, k))

    def chi2_cdf(self, x, k):
        return float(self.f("chi2_cdf")(x, k))

    def chi2_quantile(self, a, k):
        return float(self.f("chi2_quantile")(a, k))

    # ---- stages --------------------------------------------------------------
    def sample_hash_family(self, d, K, L, seed):
        out = np.empty((L, K, d), np.float32)
        self.f("sample_hash_family")(d, K, L, seed, _p(out))
        return out

    def project_dataset(self, coeffs, data):
        L, K, d = coeffs.shape
        data = np.ascontiguousarray(data, np.float32)
        coeffs = np.ascontiguousarray(coeffs, np.float32)
        out = np.empty((L, data.shape[0], K), np.float32)
        self.f("project_dataset")(_p(coeffs), K, L, _p(data), data.shape[0], d, _p(out))
        return out

    def select_breakpoints(self, proj, n_regions, sample_fraction, seed, want_idx=False):
        L, n, K = proj.shape
        proj = np.ascontiguousarray(proj, np.float32)
        out = np.empty((L, K, n_regions + 1), np.float32)
        ns = C.c_uint64(0)
        if self.kind == "port":
            n_s = max(int(np.ceil(sample_fraction * n)), n_regions)
            idx = np.empty((L, n_s), np.uint64) if want_idx else None
            draws = np.empty(L * K, np.uint64)
            rc = self.f("select_breakpoints")(_p(proj), n, K, L, n_regions, sample_fraction, seed,
                                              _p(out), C.byref(ns),
                                              _p(idx) if want_idx else None, _p(draws))
            assert rc == 0
            return (out, int(ns.value), idx, draws) if want_idx else out
        rc = self.f("select_breakpoints")(_p(proj), n, K, L, n_regions, sample_fraction, seed,
                                          _p(out), C.byref(ns))
        assert rc == 0, self.lib.ref_last_error()
        return out

    def select_row_breakpoints(self, sample, n_regions, rng_seed):
        s = np.array(sample, np.float32)
        out = np.empty(n_regions + 1, np.float32)
        if self.kind == "port":
            rng = C.create_string_buffer(312 * 8 + 64)
            self.lib.orc_rng_seed(rng, rng_seed)
            assert self.f("select_row_breakpoints")(_p(s), len(s), n_regions, rng, _p(out)) == 0
        else:
            assert self.f("select_row_breakpoints")(_p(s), len(s), n_regions, rng_seed, _p(out)) == 0
        return out, s

    def locate_region(self, v, row):
        row = np.ascontiguousarray(row, np.float32)
        return int(self.f("locate_region")(C.c_float(v), _p(row), len(row) - 1))

    def encode_dataset(self, proj, table):
        L, n, K = proj.shape
        proj = np.ascontiguousarray(proj, np.float32)
        table = np.ascontiguousarray(table, np.float32)
        out = np.empty((L, n, K), np.uint8)
        self.f("encode_dataset")(_p(proj), n, K, L, _p(table), table.shape[2] - 1, _p(out))
        return out

    def build_tree(self, codes, n_regions, space, max_size):
        L, n, K = codes.shape
        codes = np.ascontiguousarray(codes, np.uint8)
        h = self.f("build_tree")(_p(codes), n, K, L, n_regions, space, max_size)
        assert h
        return OracleTree(self, h, K, n)

    def build_index(self, data, params: Params, seed: int, table=None):
        data = np.ascontiguousarray(data, np.float32)
        n, d = data.shape
        p = Params.from_buffer_copy(params)
        if table is None:
            if self.kind == "port":
                h = self.f("build_index")(_p(data), n, d, C.byref(p), seed)
            else:
                secs = C.c_double(0)
                h = self.f("build_index")(_p(data), n, d, C.byref(p), seed, C.byref(secs))
        else:
            table = np.ascontiguousarray(table, np.float32)
            if self.kind == "port":
                h = self.f("build_index_with_table")(_p(data), n, d, C.byref(p), seed, _p(table))
            else:
                n_s = max(int(np.ceil(p.sample_fraction * n)), p.n_regions)
                h = self.f("build_index_with_table")(_p(data), n, d, C.byref(p), seed, _p(table), n_s)
        assert h, "oracle build failed"
        return OracleIndex(self, h, p, data)

    def build_det_only_index(self, data, params: Params, seed: int):
        """Reference only: detlsh::build_det_only_index (index.cpp:220-232)."""
        data = np.ascontiguousarray(data, np.float32)
        p = Params.from_buffer_copy(params)
        h = self.f("build_det_only_index")(_p(data), data.shape[0], data.shape[1], C.byref(p), seed)
        assert h, "reference det-only build failed"
        return OracleIndex(self, h, p, data)

    def load_index(self, blob: bytes, data, params: Params):
        """Reference only: detlsh::load_index (persist.cpp:157-246) of DETL v1 bytes."""
        data = np.ascontiguousarray(data, np.float32)
        buf = np.frombuffer(blob, np.uint8)
        h = self.f("index_load")(_p(buf), len(blob), _p(data), data.shape[0], data.shape[1])
        return OracleIndex(self, h, params, data) if h else None

    def brute_force_knn(self, data, Q, k):
        data = np.ascontiguousarray(data, np.float32)
        Q = np.ascontiguousarray(Q, np.float32)
        ids = np.empty((Q.shape[0], k), np.uint32)
        ds = np.empty((Q.shape[0], k), np.float64)
        self.f("brute_force_knn")(_p(data), data.shape[0], data.shape[1], _p(Q), Q.shape[0], k,
                                  _p(ids), _p(ds))
        return ids, ds


def _export(lib_fn, handle_args, K, nn, n_entries):
    rc = np.empty(1 << K, np.int32)
    out = TreeExport(rc, np.empty(nn, np.uint8), np.empty(nn, np.uint8), np.empty(nn, np.int32),
                     np.empty(nn, np.int32), np.empty((nn, K), np.uint8),
                     np.empty((nn, K), np.uint8), np.empty(nn, np.uint64),
                     np.empty(nn, np.uint32), np.empty(n_entries, np.uint32))
    lib_fn(*handle_args, _p(out.root_children), _p(out.is_leaf), _p(out.split_dim), _p(out.left),
           _p(out.right), _p(out.bits), _p(out.value), _p(out.ebegin), _p(out.ecount),
           _p(out.positions))
    return out


class OracleTree:
    def __init__(self, orc: Oracle, h, K, n):
        self.o, self.h, self.K, self.n = orc, h, K, n

    def __del__(self):
        try:
            self.o.f("tree_free")(self.h)
        except Exception:
            pass

    def export(self) -> TreeExport:
        nn = int(self.o.f("tree_num_nodes")(self.h))
        return _export(self.o.f("tree_export"), (self.h,), self.K, nn, self.n)

    def range_query_optimized(self, table, q_proj, radius, limit):
        table = np.ascontiguousarray(table, np.float32)
        q = np.ascontiguousarray(q_proj, np.float32)
        out = np.empty(max(1, min(limit, self.n)), np.uint32)
        if self.o.kind == "port":
            cnt = self.o.f("range_query_optimized")(self.h, _p(table), _p(q), radius, limit, _p(out))
        else:
            cnt = self.o.f("range_query_optimized")(self.h, _p(table), table.shape[2] - 1, _p(q),
                                                    radius, limit, _p(out))
        return out[:cnt].copy()


class OracleIndex:
    def __init__(self, orc: Oracle, h, params: Params, data):
        self.o, self.h, self.params, self.data = orc, h, params, data

    def __del__(self):
        try:
            self.o.f("index_free")(self.h)
        except Exception:
            pass

    @property
    def n(self):
        return self.data.shape[0]

    @property
    def d(self):
        return self.data.shape[1]

    def table(self):
        p = self.params
        out = np.empty((p.L, p.K, p.n_regions + 1), np.float32)
        self.o.f("index_table")(self.h, _p(out))
        return out

    def tree_export(self, i) -> TreeExport:
        if self.o.kind != "port":
            nn = int(self.o.f("index_tree_nodes")(self.h, i))
            return _export(self.o.f("index_tree_export"), (self.h, i), self.params.K, nn, self.n)
        tptr = self.o.lib.orc_index_tree
        tptr.argtypes, tptr.restype = [C.c_void_p, C.c_int], C.c_void_p
        t = tptr(self.h, i)
        nn = int(self.o.f("tree_num_nodes")(t))
        return _export(self.o.f("tree_export"), (t,), self.params.K, nn, self.n)

    def rc_ann(self, q, r, c):
        """Reference only: detlsh::rc_ann -> (pos, dist) or None."""
        q = np.ascontiguousarray(q, np.float32)
        pos = C.c_uint32(0)
        dist = C.c_double(0)
        rc = self.o.f("rc_ann")(self.h, _p(q), r, c, C.byref(pos), C.byref(dist))
        assert rc >= 0
        return (pos.value, dist.value) if rc == 1 else None

    def estimate_rmin(self, probes, k):
        """Reference only: detlsh::estimate_rmin (index.cpp:333-374)."""
        P = np.ascontiguousarray(probes, np.float32)
        return float(self.o.f("index_estimate_rmin")(self.h, _p(P), P.shape[0], k))

    def project_query(self, q, space):
        """Reference only: DetIndex::project_query (index.cpp:181-188)."""
        q = np.ascontiguousarray(q, np.float32)
        out = np.empty(self.params.K, np.float32)
        self.o.f("index_project_query")(self.h, _p(q), space, _p(out))
        return out

    def range_query(self, tree, q_proj, radius, limit=2**63, exact=False):
        """Reference only: range_query_optimized (sink stops after `limit`) or
        range_query_exact on tree `tree` (de_tree.cpp:199-258)."""
        q = np.ascontiguousarray(q_proj, np.float32)
        cap = min(self.n, limit)
        out = np.empty(max(1, cap), np.uint32)
        m = int(self.o.f("index_range_query")(self.h, tree, _p(q), radius, limit, int(exact), _p(out), cap))
        return out[:min(m, cap)].copy()

    def save(self) -> bytes:
        """Reference only: detlsh::save_index (persist.cpp:99-149) bytes."""
        size = int(self.o.f("index_save")(self.h, None, 0))
        buf = np.empty(size, np.uint8)
        self.o.f("index_save")(self.h, _p(buf), size)
        return buf.tobytes()

    def ck_ann(self, q, k):
        q = np.ascontiguousarray(q, np.float32)
        ids = np.empty(k, np.uint32)
        ds = np.empty(k, np.float64)
        nh = C.c_int(0)
        rad = C.c_double(0)
        cs = C.c_uint64(0)
        rc = self.o.f("ck_ann")(self.h, _p(q), k, _p(ids), _p(ds), C.byref(nh), C.byref(rad),
                                C.byref(cs))
        assert rc == 0
        m = nh.value
        return ids[:m].copy(), ds[:m].copy(), rad.value, cs.value

    def ck_ann_batch(self, Q, k, threads=1):
        """Reference only: std::thread pool over ck_ann; returns (ids, dists, nh, rad, cands, secs)."""
        Q = np.ascontiguousarray(Q, np.float32)
        nq = Q.shape[0]
        ids = np.zeros((nq, k), np.uint32)
        ds = np.zeros((nq, k), np.float64)
        nh = np.zeros(nq, np.int32)
        rad = np.zeros(nq, np.float64)
        cs = np.zeros(nq, np.uint64)
        secs = C.c_double(0)
        if self.o.kind == "port":
            import time
            t0 = time.perf_counter()
            for i in range(nq):
                a, b, r, c = self.ck_ann(Q[i], k)
                ids[i, :len(a)] = a
                ds[i, :len(a)] = b
                nh[i], rad[i], cs[i] = len(a), r, c
            return ids, ds, nh, rad, cs, time.perf_counter() - t0
        rc = self.o.f("ck_ann_batch")(self.h, _p(Q), nq, k, threads, _p(ids), _p(ds), _p(nh),
                                      _p(rad), _p(cs), C.byref(secs))
        assert rc == 0
        return ids, ds, nh, rad, cs, secs.value
