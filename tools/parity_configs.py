"""Parity at scale: the GPU path vs the REFERENCE library (oracle/_ref, compiled
from the reference sources) on the BASELINE configs (full C1, subsets of C2-C4).
Writes a JSON summary (path from argv[1]) with per-config bit-exact counts,
recall/ratio of both, and timings.  Measurement/evidence tool, not product."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402
from oracle.bindings import Oracle, make_params, ref_available  # noqa: E402

CASES = [
    ("c1", 100_000, 1000, 1000),   # full config 1, all queries checked
    ("c2", 200_000, 200, 200),
    ("c2", 1_000_000, 2000, 300),  # full C2 index: tensor-core verification path
    ("c3", 100_000, 100, 100),
    ("c4", 1_000_000, 100, 50),
]


def main(out_path):
    ref = Oracle("reference" if ref_available() else "port")
    threads = os.cpu_count() or 1
    summary = {"oracle": ref.kind, "cases": []}
    for cfg, n, nq, ncheck in CASES:
        base, Q = gen.make(cfg, n=n, nq=nq)
        p = dict(beta=0.1, k=50)
        t0 = time.perf_counter()
        idx = D.build_index(base, D.LshParams(**p), seed=7)
        t_gpu_build = time.perf_counter() - t0
        t0 = time.perf_counter()
        res = D.ck_ann_batch(idx, Q, 50)
        t_gpu_q = time.perf_counter() - t0
        t0 = time.perf_counter()
        oi = ref.build_index(base, make_params(**p), 7)
        t_ref_build = time.perf_counter() - t0
        ids, ds, nh, rad, cs, secs = oi.ck_ann_batch(Q[:ncheck], 50, threads=threads)
        same = 0
        for i in range(ncheck):
            m = int(nh[i])
            ok = (int(res.n_hits[i]) == m and np.array_equal(res.ids[i, :m], ids[i, :m])
                  and np.array_equal(res.dists[i, :m].view(np.uint64), ds[i, :m].view(np.uint64))
                  and res.radius_used[i] == rad[i] and int(res.candidates_seen[i]) == int(cs[i]))
            same += ok
        tab = np.array_equal(idx.table().view(np.uint32), oi.table().view(np.uint32))
        case = dict(config=cfg, n=n, d=int(base.shape[1]), queries_checked=ncheck,
                    bit_exact_queries=same, table_bit_exact=bool(tab),
                    r_min_equal=bool(idx.params.r_min == oi.params.r_min),
                    gpu_build_s=round(t_gpu_build, 4), ref_build_s=round(t_ref_build, 3),
                    gpu_query_s=round(t_gpu_q, 4), ref_query_s=round(secs, 3), ref_threads=threads)
        summary["cases"].append(case)
        print(json.dumps(case), flush=True)
    with open(out_path, "w") as f:
        json.dump(summary, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "parity_configs.json")
