"""A/B of the query verification paths on a config: tcgen05 dataset-major
scoring vs the per-query gather path.  Checks the results are identical and
prints wall time per batch (host arrays, copies included) for each."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
k = int(sys.argv[3]) if len(sys.argv) > 3 else 50
beta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.1  # bench.py's beta
base, Q = gen.make(cfg, nq=nq)
idx = D.build_index(base, D.LshParams(k=k, beta=beta), seed=2, keep_codes=False)
print(f"{cfg}: n={base.shape[0]} d={base.shape[1]} nq={nq} k={k} budget={D.candidate_budget(idx.params.beta, base.shape[0], k)} row_u8={idx.row_u8()}")
res = {}
for tc in (True, False):
    D.ck_ann_batch(idx, Q, k, tensor_cores=tc)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        r = D.ck_ann_batch(idx, Q, k, tensor_cores=tc)
        ts.append(time.perf_counter() - t0)
    res[tc] = r
    t = min(ts)
    print(f"  tensor_cores={tc!s:5s}: {1e3 * t:8.2f} ms/batch  {nq / t:10.0f} q/s")
    lib = D.load()
    lib.detlsh_profile_enable(1)
    D.ck_ann_batch(idx, Q, k, tensor_cores=tc)
    lib.detlsh_profile_enable(0)
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
    for i, name in enumerate(names.value.decode().split(";")[:m]):
        print(f"      {name:20s} {ms[i]:8.3f} ms  x{int(cnt[i])}")
a, b = res[True], res[False]
same = (np.array_equal(a.ids, b.ids) and np.array_equal(a.dists.view(np.uint64), b.dists.view(np.uint64))
        and np.array_equal(a.n_hits, b.n_hits))
print(f"  identical results: {same}")
if not same:
    bad = np.nonzero((a.ids != b.ids).any(1) | (a.n_hits != b.n_hits))[0]
    print(f"  mismatching queries: {len(bad)} first {bad[:10].tolist()}")
    sys.exit(1)
