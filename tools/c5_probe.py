"""C5 (1e8 x 128) feasibility probe on one B200: device-generated data, build
(GPU-native sample by default), a query batch, memory high-water marks."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402


def mem():
    f, t = torch.cuda.mem_get_info()
    return round((t - f) / 2**30, 2)


ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000_000)
ap.add_argument("--nq", type=int, default=1000)
ap.add_argument("--sample", default="gpu")
ap.add_argument("--builds", type=int, default=2)
ap.add_argument("--tau", default="", help="comma list of DETLSH_TAU_ROWS values to sweep")
a = ap.parse_args()
t0 = time.time()
base, Q = gen.make_device("c5", n=a.n, nq=a.nq)
torch.cuda.synchronize()
out = {"n": a.n, "nq": a.nq, "gen_s": round(time.time() - t0, 2), "mem_after_gen_gb": mem()}
p = D.LshParams(beta=0.1, k=50)
for b in range(a.builds):
    t0 = time.time()
    idx = D.build_index(base, p, seed=5, sample=a.sample, borrow=True, keep_codes=False)
    torch.cuda.synchronize()
    out[f"build{b}_s"] = round(time.time() - t0, 3)
    out["mem_after_build_gb"] = mem()
    if b + 1 < a.builds:
        del idx
out["stages"] = idx.build_timings()
out["r_min"] = idx.params.r_min
out["row_u8"] = idx.row_u8()
print(json.dumps(out), flush=True)
k = 50
ids = torch.empty((a.nq, k), dtype=torch.int32, device="cuda")
ds = torch.empty((a.nq, k), dtype=torch.float64, device="cuda")
nh = torch.empty(a.nq, dtype=torch.int32, device="cuda")
lib = D.load()
import ctypes as C  # noqa: E402
for tau in (a.tau.split(",") if a.tau else [""]):
    if tau:
        os.environ["DETLSH_TAU_ROWS"] = tau
    res = {"tau_rows": tau or "default"}
    for rep in range(2):
        torch.cuda.synchronize()
        if rep == 0:
            os.environ["DETLSH_DEBUG_QUERY"] = "1"
        else:
            os.environ.pop("DETLSH_DEBUG_QUERY", None)
            lib.detlsh_profile_enable(1)
        t0 = time.time()
        D.ck_ann_device(idx, Q, k, ids, ds, nh)
        torch.cuda.synchronize()
        res[f"query{rep}_s"] = round(time.time() - t0, 3)
    lib.detlsh_profile_enable(0)
    if os.environ.get("C5_SLOW_PHASES"):  # one more batch with the general-path phase split on stderr
        os.environ["DETLSH_DEBUG_QUERY"] = "1"
        lib.detlsh_profile_enable(1)
        D.ck_ann_device(idx, Q, k, ids, ds, nh)
        torch.cuda.synchronize()
        lib.detlsh_profile_enable(0)
        os.environ.pop("DETLSH_DEBUG_QUERY", None)
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
    res["query_kernels_ms"] = {kk: round(float(ms[i]), 3) for i, kk in enumerate(names.value.decode().split(";")[:m])}
    ph = np.zeros(8)
    lib.detlsh_query_phase_cycles(C.c_void_p(ph.ctypes.data))
    res["phase_kcycles_per_query"] = [round(v / a.nq / 1e3, 1) for v in ph[:6]]
    res["qps"] = round(a.nq / res["query1_s"], 1)
    res["hits_min"] = int(nh.min().item())
    res["ids_sum"] = int(ids.to(torch.int64).sum().item())
    print(json.dumps(res), flush=True)
print(json.dumps({"mem_after_query_gb": mem()}), flush=True)
