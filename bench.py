#!/usr/bin/env python
"""DET-LSH on B200: index build (Mpoints/s) + batched 50-NN queries (queries/s).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload: BASELINE.json configs[1] ("c2": n=1e6, d=128 sparse 8-bit integers,
10,000 held-out queries, K=16, L=4, N_r=256, leaf 128, k=50, c=1.5, beta=0.1),
synthetic (paper_2406_10938_b200/data.py).  One build step = build_index over
the whole (per-rank) shard; one query step = the whole 10,000-query batch
through ck_ann, merged across ranks.  `value` is the build rate; the query
rate, recall and ratio are in "query".  Multi-GPU: point-sharded independent
indexes, NCCL all-gather of per-shard top-k + GPU merge.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DE-Tree index build Mpoints/s; batched 50-NN queries/s at reference-matched recall"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--nq", type=int, default=None)
    ap.add_argument("--k", type=int, default=50)
    ap.add_argument("--beta", type=float, default=0.1)
    ap.add_argument("--seed", type=int, default=2)
    ap.add_argument("--sample", choices=["reference", "gpu"], default="reference",
                    help="breakpoint sample mode of the headline build")
    ap.add_argument("--shard", choices=["weak", "strong"], default="strong",
                    help="N>1: strong (default, BASELINE configs 4-5) = the config's one n-point "
                         "dataset split into N contiguous point shards; weak = every rank indexes "
                         "its own n-point shard of a world x n dataset (fixed per-GPU work)")
    ap.add_argument("--plumbing", action="store_true",
                    help="check the multi-rank launch only (no GPU needed): ranks, shard bounds, "
                         "the all-gather of per-shard lists; rank 0 prints one JSON line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-queries", type=int, default=200)
    ap.add_argument("--gt-queries", type=int, default=500,
                    help="c5: queries scored against the exact kNN (device brute force)")
    ap.add_argument("--cpu-build-rows", type=int, default=None,
                    help="rows the reference build is timed on (default: the full n, same config)")
    return ap.parse_args()


def relaunch_distributed(args):
    """`bench.py --gpus N` without a torchrun environment: re-exec under
    torch.distributed.run with N ranks on this node (one process per GPU)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


# ---------------------------------------------------------------------------
# clocks sampled with nvidia-smi during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        # in-process NVML sampling (a light query every 100 ms); the nvidia-smi
        # loop is the fallback (its driver calls can stall a host-sync-heavy build)
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.stop_flag = False
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _poll(self):
        nv = self.nvml
        bits = [("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
                ("sw_power_cap", 0x4)]
        while not self.stop_flag:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM)
                mx = nv.nvmlDeviceGetMaxClockInfo(self.handle, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle)
                self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for _, b in bits])
            except Exception:
                pass
            time.sleep(0.1)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if getattr(self, "nvml", None) is not None:
            time.sleep(0.15)
            self.stop_flag = True
            self.thread.join(timeout=2)
        elif self.proc is None:
            return None
        else:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# ground truth + quality metrics (measurement only, outside the timed region)
# ---------------------------------------------------------------------------
def exact_knn_gpu(base, Q, k, integer_data: bool):
    """metrics.cpp:8-33 semantics: order by (dist^2, position)."""
    import torch
    torch.backends.cuda.matmul.allow_tf32 = False
    dt = torch.float32 if integer_data else torch.float64
    X = torch.from_numpy(base).cuda().to(dt)
    xn = (X * X).sum(1)
    ids = np.empty((Q.shape[0], k), np.int64)
    dists = np.empty((Q.shape[0], k), np.float64)
    step = 256
    for s in range(0, Q.shape[0], step):
        q = torch.from_numpy(Q[s:s + step]).cuda().to(dt)
        D = (q * q).sum(1, keepdim=True) + xn[None, :] - 2.0 * (q @ X.T)
        if integer_data:
            D = torch.round(D)
        D = D.clamp_min_(0)
        kth = torch.kthvalue(D, k, dim=1).values
        for i in range(q.shape[0]):
            row = D[i]
            t = kth[i]
            less = torch.nonzero(row < t).flatten()
            lv = row[less]
            order = torch.argsort(lv, stable=True)  # positions ascending within ties
            less = less[order]
            eq = torch.nonzero(row == t).flatten()[: k - less.numel()]
            sel = torch.cat([less, eq])
            ids[s + i] = sel.cpu().numpy()
            dists[s + i] = np.sqrt(row[sel].double().cpu().numpy())
    return ids, dists


def recall_ratio(res_ids, res_d, n_hits, gt_ids, gt_d, k):
    """recall / overall_ratio as metrics.cpp:35-66."""
    rec, rat = [], []
    for i in range(res_ids.shape[0]):
        m = int(n_hits[i])
        rec.append(len(set(res_ids[i, :m].tolist()) & set(gt_ids[i].tolist())) / k)
        s, cnt = 0.0, 0
        for r in range(min(m, k)):
            t, v = gt_d[i, r], res_d[i, r]
            if t == 0.0:
                if v == 0.0:
                    s += 1.0
                    cnt += 1
                continue
            s += v / t
            cnt += 1
        rat.append(1.0 if cnt == 0 else s / cnt)
    return float(np.mean(rec)), float(np.mean(rat))


def tc_tau_rows(k, budget, R=128):
    """Rows the plan kernel scores exactly for tau^2 (query.cu run_query_batch):
    the staging cap is 16 K for rows wider than 256 B or budgets of 2^20+, else 4 K."""
    cap = 16384 if (R > 256 or budget >= (1 << 20)) else 4096
    return max(512, 2 * k, min((1 << 17) * 4096 // cap, -(-4 * k * budget // cap)))  # kTauRowsMax


# algorithmic bytes per launch; kernels without a model get null
def algo_bytes(kernel, n, d, nq, budget, K, L, row_u8=0, plan=None):
    if kernel in ("project_exact", "project_tc"):
        return 4.0 * d * n  # one read of the fp32 shard (4d B/point)
    if kernel == "query_fast" and plan is not None:
        # tensor-core hand-off: per query the plan kernel reads tree 0's 8-byte
        # leaf records, writes and re-reads a 2-byte bin per leaf, scores
        # tau_rows u8 rows and writes the n-bit candidate row bitmap
        return (12.0 * plan["leaves"] + row_u8 * plan["tau_rows"] + n / 8.0) * nq
    if kernel == "query_fast":
        return 4.0 * d * budget * nq  # every verified candidate row (4d B/candidate)
    if kernel == "encode":
        return 5.0 * K * n  # one space per launch: fp32 projections in, u8 codes out
    if kernel == "tree_sort":
        return (K + 4.0) * n  # one tree: read its codes, write the leaf-order permutation
    if kernel == "rmin_dist":
        return (4.0 * L * K + 8.0 * 10) * n  # read projections, write 10 probe distances
    if kernel == "pack_u8":
        return (4.0 * d + ((d + 31) // 32 * 32)) * n  # gathered fp32 rows in, u8 rows out
    return None


def ncu_traffic(kernel, units, cfg_key):
    """dram__bytes_read+write for `kernel` from the committed ncu capture
    (profiles/ncu_latest.json), only when that capture ran this same config
    (`cfg_key`, e.g. "c2:n=1000000:nq=10000"); otherwise null."""
    path = os.path.join(ROOT, "profiles", "ncu_latest.json")
    try:
        with open(path) as f:
            table = json.load(f)
        recs = table.get(kernel) or table[kernel + "_kernel"]  # {config: record}
        rec = recs.get(cfg_key)
        if rec is None:
            return None, None
        return rec["dram_bytes_per_unit"] * units, rec["source"]
    except Exception:
        return None, None


OWN_PEAKS_PATH = os.path.join(ROOT, "profiles", "peaks_measured.json")


def own_peaks():
    """FP64-DMMA and tcgen05 kind::i8 peaks measured on a B200 of this pool by
    tools/probes/peaks.cu (committed JSON), or None."""
    try:
        with open(OWN_PEAKS_PATH) as f:
            return json.load(f)
    except Exception:
        return None


def peak_bf16():
    try:
        with open(PEAKS_PATH) as f:
            return float(json.load(f)["bf16_tflops"])
    except Exception:
        return 2250.0


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# the reference arm: the reference's own CPU implementation
# ---------------------------------------------------------------------------
def run_reference(args, rank):
    if rank != 0:
        return
    from oracle.bindings import Oracle, ref_available, make_params
    from paper_2406_10938_b200 import data as gen
    kind = "reference" if ref_available() else "port"
    orc = Oracle(kind)
    cfg = args.config
    base, Q = gen.make(cfg, nq=args.nq)
    n, d = base.shape
    cores = os.cpu_count() or 1
    p = make_params(beta=args.beta, k=args.k)
    rows = n if args.cpu_build_rows is None else min(n, args.cpu_build_rows)
    sub = np.ascontiguousarray(base[:rows])
    # build: single thread (the reference is single-threaded by design)
    times = []
    full = None
    for step in range(args.warmup + args.steps):
        full = None  # one index alive at a time
        t0 = time.perf_counter()
        full = orc.build_index(sub, p, args.seed)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(dt)
    build_s = float(np.mean(times))
    build_rate = rows / build_s / 1e6
    # queries: full-size index (the last timed build when it covered all n), all host threads
    if rows != n:
        full = None
        full = orc.build_index(base, p, args.seed)
    nqs = min(args.cpu_queries, Q.shape[0])
    qtimes = []
    for step in range(args.warmup + args.steps):
        qs = Q[(step * nqs) % Q.shape[0]:][:nqs]
        ids, ds, nh, rad, cs, secs = full.ck_ann_batch(qs, args.k, threads=cores)
        if step >= args.warmup:
            qtimes.append(secs)
    q_rate = nqs / float(np.mean(qtimes))
    integer = bool(np.all(base == np.round(base)) and base.min() >= 0 and base.max() <= 255)
    gt_ids, gt_d = exact_knn_gpu_or_cpu(base, Q[:nqs], args.k, integer, orc)
    ids, ds, nh, rad, cs, _ = full.ck_ann_batch(Q[:nqs], args.k, threads=cores)
    rec, rat = recall_ratio(ids, ds, nh, gt_ids, gt_d, args.k)
    sample = (f"build: {'all' if rows == n else 'first'} {rows} of {n} rows x {args.steps} steps, 1 thread; "
              f"queries: {nqs} per step on the full n={n} index, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(build_rate, 6), "unit": "Mpoints/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(build_s * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg}: n={n}, d={d}, nq={Q.shape[0]}, K=16, L=4, N_r=256, "
                               f"leaf=128, k={args.k}, c=1.5, beta={args.beta}",
                   "parallelism": "cpu"},
        "query": {"value": round(q_rate, 3), "unit": "queries/s", "recall": rec, "ratio": rat,
                  "queries": nqs},
        "cpu_baseline": {"value": round(build_rate, 6), "unit": "Mpoints/s", "cores": 1,
                         "kind": kind, "sample": sample,
                         "query": {"value": round(q_rate, 3), "unit": "queries/s",
                                   "cores": cores}},
        "e2e": {"value": round(build_rate, 6), "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def exact_knn_gpu_or_cpu(base, Q, k, integer, orc):
    try:
        import torch
        if torch.cuda.is_available():
            return exact_knn_gpu(base, Q, k, integer)
    except Exception:
        pass
    return orc.brute_force_knn(base, Q, k)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def cpu_baseline(args, base, Q):
    """The reference (oracle/_ref) on this box's host cores, bounded sample."""
    from oracle.bindings import Oracle, ref_available, make_params
    kind = "reference" if ref_available() else "port"
    orc = Oracle(kind)
    n = base.shape[0]
    rows = n if args.cpu_build_rows is None else min(n, args.cpu_build_rows)
    p = make_params(beta=args.beta, k=args.k)
    t0 = time.perf_counter()
    full = orc.build_index(np.ascontiguousarray(base[:rows]), p, args.seed)
    b = time.perf_counter() - t0
    if rows != n:
        full = orc.build_index(base, p, args.seed)
    cores = os.cpu_count() or 1
    nqs = min(args.cpu_queries, Q.shape[0])
    _, _, _, _, _, secs = full.ck_ann_batch(Q[:nqs], args.k, threads=cores)
    return {"value": round(rows / b / 1e6, 6), "unit": "Mpoints/s", "cores": 1, "kind": kind,
            "sample": f"build_index on {'all' if rows == n else 'the first'} {rows} rows (1 thread); ck_ann on {nqs} "
                      f"queries against the full n={n} index ({cores} threads)",
            "query": {"value": round(nqs / secs, 3), "unit": "queries/s", "cores": cores}}


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args)  # does not return
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.plumbing:
        plumbing(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank)
        return

    import torch
    import torch.distributed as dist
    import paper_2406_10938_b200 as D
    from paper_2406_10938_b200 import data as gen
    from paper_2406_10938_b200.shard import gather_topk, shard_bounds

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = D.load()
    cfg = args.config
    devgen = cfg == "c5"  # 51 GB: generated on the GPU, never through host memory
    if devgen:
        base_d, Q_d = gen.make_device(cfg, nq=args.nq, device=local)
        base = None
        Q = Q_d.cpu().numpy()
        n, d = base_d.shape
    else:
        base, Q = gen.make(cfg, nq=args.nq)
        n, d = base.shape
    nq = Q.shape[0]
    if devgen:
        if world > 1 and args.shard == "weak":
            raise SystemExit("c5: strong (point-sharded) scaling only")
        s0, s1 = shard_bounds(n, world, rank)
        shard = None
        n_total = n
    elif world > 1 and args.shard == "weak":
        # weak scaling: rank r holds points [r n, (r+1) n) of a world x n dataset
        shard = base if rank == 0 else np.ascontiguousarray(gen.make_shard(cfg, rank, n))
        s0 = rank * n
        n_total = world * n
    else:
        s0, s1 = shard_bounds(n, world, rank)
        shard = np.ascontiguousarray(base[s0:s1])
        n_total = n
    n_loc = (s1 - s0) if devgen else shard.shape[0]
    params = D.LshParams(beta=args.beta, k=args.k)
    k = args.k
    dev_shard = base_d[s0:s1] if devgen else torch.from_numpy(shard).cuda()
    dev_Q = Q_d if devgen else torch.from_numpy(Q).cuda()
    # page-locked host copies for the end-to-end legs, made here, long before
    # they are timed (pinning 0.5 GB on a fresh box leaves the host busy for a
    # while: the first end-to-end builds after it ran 47-62 ms instead of 33)
    shard_pinned = None if devgen else torch.from_numpy(shard).pin_memory().numpy()
    Qpin = torch.from_numpy(Q).pin_memory().numpy()
    # a stream of our own: the queries are enqueued on it (device mode returns
    # at once) and the timing events are recorded on it, so they bracket the
    # kernels (the legacy default stream would not order the library's streams)
    stream = torch.cuda.Stream()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps):
        gc.collect()  # indexes left in reference cycles by earlier phases
        return _timed(fn, steps)

    def _timed(fn, steps):
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        out = None
        walls = []
        for _ in range(steps):
            w0 = time.perf_counter()
            out = fn()
            walls.append((time.perf_counter() - w0) * 1e3)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        print(f"[bench] {getattr(fn, '__name__', 'step')}: host ms per step " +
              " ".join(f"{w:.2f}" for w in walls), file=sys.stderr)
        return e0.elapsed_time(e1) / steps, out

    # ---------------- build ----------------
    def build():
        return D.build_index(dev_shard, params, seed=args.seed, sample=args.sample, borrow=True,
                             keep_codes=False)

    # the GPU-native breakpoint sample, reported beside the headline
    # (timed first: no headline index is alive yet, as in the headline's own loop)
    other = "gpu" if args.sample == "reference" else "reference"

    def build_other():
        return D.build_index(dev_shard, params, seed=args.seed, sample=other, borrow=True,
                             keep_codes=False)

    w = None
    for _ in range(args.warmup):  # same live-index pattern as the timed loop
        w = build_other()
    del w
    other_ms, other_idx = timed(build_other, args.steps)
    other_stages = other_idx.build_timings()
    del other_idx
    other_ms = max_over_ranks(other_ms)

    # The timed steps run without the per-kernel event profile (its phase
    # read-backs are host waits that would open gaps between batches); the
    # profile comes from as many extra steps of the same workload right after.
    for _ in range(args.warmup):
        idx = build()
    del idx
    clocks = ClockSampler(local)
    clocks.start()
    lc0 = lib.detlsh_launch_count()
    build_ms, idx = timed(build, args.steps)
    build_launches = (lib.detlsh_launch_count() - lc0) / args.steps
    build_ms = max_over_ranks(build_ms)
    stage_ms = idx.build_timings()
    prof_build = profiled_steps(lib, build, args.steps)

    # ---------------- queries ----------------
    ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    dists = torch.empty((nq, k), dtype=torch.float64, device="cuda")
    hits = torch.empty(nq, dtype=torch.int32, device="cuda")
    rad = torch.empty(nq, dtype=torch.float64, device="cuda")
    cands = torch.empty(nq, dtype=torch.int64, device="cuda")
    if world > 1:
        g_d = torch.empty((world, nq, k), dtype=torch.float64, device="cuda")
        g_i = torch.empty((world, nq, k), dtype=torch.int64, device="cuda")
        g_h = torch.empty((world, nq), dtype=torch.int32, device="cuda")
        m_d = torch.empty((nq, k), dtype=torch.float64, device="cuda")
        m_i = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        m_h = torch.empty(nq, dtype=torch.int32, device="cuda")

    def query():
        D.ck_ann_device(idx, dev_Q, k, ids, dists, hits, rad, cands, stream=stream.cuda_stream)
        if world == 1:
            return ids, dists, hits
        with torch.cuda.stream(stream):  # the exchange is ordered after the batch
            gid = ids.to(torch.int64) + s0  # global positions
            gather_topk(dists, gid, hits, g_d, g_i, g_h)
            D.merge_topk_device(g_d, g_i, g_h, k, m_d, m_i, m_h, stream=stream.cuda_stream)
        return m_i, m_d, m_h

    for _ in range(args.warmup):
        query()
    lc0 = lib.detlsh_launch_count()
    query_ms, (r_ids, r_d, r_h) = timed(query, args.steps)
    query_launches = (lib.detlsh_launch_count() - lc0) / args.steps
    query_ms = max_over_ranks(query_ms)
    clk = clocks.stop()
    prof_query = profiled_steps(lib, query, args.steps)

    # ---------------- end to end through the public API, host buffers ----------------

    def e2e_build():
        ix = D.build_index(shard_pinned, params, seed=args.seed, device=local, sample=args.sample,
                           keep_codes=False)
        _ = ix.params.r_min  # result read back (params travel D2H inside build)
        return ix

    e2e_build_ms = None
    if not devgen:  # (c5's 51 GB shard lives on the device only)
        w = None
        for _ in range(args.warmup):  # same live-index pattern as the timed loop
            w = e2e_build()
        del w
        e2e_build_ms, ix2 = timed(e2e_build, max(1, args.steps))
        e2e_build_ms = max_over_ranks(e2e_build_ms)
        del ix2

    # page-locked result arrays, reused across steps (what a serving loop does)
    def pinned(shape, dt):
        return torch.empty(shape, dtype=dt, pin_memory=True).numpy()

    res_pin = D.BatchResult(pinned((nq, k), torch.int32).view(np.uint32), pinned((nq, k), torch.float64),
                            pinned((nq,), torch.int32), pinned((nq,), torch.float64),
                            pinned((nq,), torch.int64).view(np.uint64))

    def e2e_query():
        res = D.ck_ann_batch(idx, Qpin, k, out=res_pin)
        if world > 1:
            t = torch.from_numpy(res.ids.astype(np.int64) + s0).cuda()
            td = torch.from_numpy(res.dists).cuda()
            th = torch.from_numpy(res.n_hits).cuda()
            gather_topk(td, t, th, g_d, g_i, g_h)
            D.merge_topk_device(g_d, g_i, g_h, k, m_d, m_i, m_h, stream=stream.cuda_stream)
            return m_i.cpu().numpy(), m_d.cpu().numpy()
        return res.ids, res.dists

    for _ in range(args.warmup):
        e2e_query()
    e2e_query_ms, _ = timed(e2e_query, max(1, args.steps))
    e2e_query_ms = max_over_ranks(e2e_query_ms)

    # ---------------- quality (merged results vs exact kNN) ----------------
    out_ids = r_ids.cpu().numpy().astype(np.int64)
    out_d = r_d.cpu().numpy()
    out_h = r_h.cpu().numpy()
    # exact ground truth with the library's brute_force_knn (metrics.cpp:8-33
    # semantics); the squared k-th returned distance bounds each query's search.
    # N > 1: every rank's exact list over its own shard, merged like the ANN lists
    # (the global exact top-k is contained in the union of the shard top-k's).
    bound = np.where(out_h == k, out_d[:, k - 1] ** 2 * (1 + 1e-12), np.inf)
    if world > 1:
        bound = None  # a shard may hold fewer than k points inside the global bound
    if devgen:  # exact kNN on the device, for the first gt_queries queries
        m_gt = min(nq, args.gt_queries)
        gi, gdd = D.brute_force_knn_device(dev_shard, dev_Q[:m_gt].contiguous(), k,
                                           dist2_bound=None if bound is None else bound[:m_gt])
        gt_ids, gt_d = gi.cpu().numpy().view(np.uint32), gdd.cpu().numpy()
        out_ids, out_d, out_h = out_ids[:m_gt], out_d[:m_gt], out_h[:m_gt]
    else:
        gt_ids, gt_d = D.brute_force_knn(shard, Q, k, dist2_bound=bound, device=local)
    gt_ids = gt_ids.astype(np.int64) + s0
    if world > 1:
        t_i = torch.from_numpy(gt_ids).cuda()
        t_d = torch.from_numpy(np.ascontiguousarray(gt_d, np.float64)).cuda()
        t_h = torch.full((nq,), min(k, n_loc), dtype=torch.int32, device="cuda")
        gather_topk(t_d, t_i, t_h, g_d, g_i, g_h)
        D.merge_topk_device(g_d, g_i, g_h, k, m_d, m_i, m_h, stream=stream.cuda_stream)
        torch.cuda.synchronize()
        gt_ids, gt_d = m_i.cpu().numpy().astype(np.int64), m_d.cpu().numpy()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    rec, rat = recall_ratio(out_ids, out_d, out_h, gt_ids, gt_d, k)

    budget = D.candidate_budget(idx.params.beta, n_loc, k)
    hbm, peak_kind = peaks()
    # candidates are single kernels: `rmin_select` and the `tree_*` scopes time
    # loops of small kernels with host reads between them, not one kernel
    cfg_key = f"{cfg}:n={n_loc}:nq={nq}"
    # the build's algorithmic bytes are one read of the fp32
    # dataset (4 d per point); the kernel that makes that read is the
    # projection, so the headline build roofline is the projection's.  The
    # other single-kernel build stages are listed with their own byte models.
    build_roof = roofline(prof_build, args.steps, n_loc, d, nq, budget, 16, 4, hbm, peak_kind,
                          only=("project_exact", "project_tc"), cfg_key=cfg_key)
    build_roof_other = {}
    for kk in ("rmin_dist", "encode", "pack_u8"):
        if kk in prof_build:
            rr = roofline(prof_build, args.steps, n_loc, d, nq, budget, 16, 4, hbm, peak_kind, only=(kk,),
                          cfg_key=cfg_key)
            if rr and rr.get("frac") is not None:
                build_roof_other[kk] = {"launch_ms": rr["launch_ms"], "achieved_gbs": rr["achieved"],
                                        "frac": rr["frac"], "algorithmic_bytes": rr.get("algorithmic_bytes")}
    build_roof_proj = None
    if "project_tc" in prof_build:  # 8-bit-integer data: tcgen05 kind::i8 over coefficient digits
        pms = prof_build["project_tc"][0] / max(1, prof_build["project_tc"][1])
        ops = 2.0 * n_loc * 5 * 64 * ((d + 31) // 32 * 32)  # 5 digit planes x 64 outputs x R
        op = own_peaks() or {}
        pk = float(op.get("int8_tcgen05_tops", 2.0 * peak_bf16()))
        build_roof_proj = {"kernel": "project_tc", "bound": "tensor (tcgen05 kind::i8)", "unit": "TOPS",
                           "achieved": round(ops / (pms / 1e3) / 1e12, 2), "peak": pk,
                           "peak_kind": ("measured (profiles/peaks_measured.json)" if "int8_tcgen05_tops" in op
                                         else "2x measured bf16 burst"),
                           "frac": round(ops / (pms / 1e3) / 1e12 / pk, 4), "launch_ms": round(pms, 4),
                           "note": "the projection of 8-bit data is HBM/epilogue bound; see roofline"}
    plan = {"leaves": int(idx.tree(0).is_leaf.sum()), "tau_rows": tc_tau_rows(k, budget, idx.row_u8())}
    query_roof = roofline(prof_query, args.steps, n_loc, d, nq, budget, 16, 4, hbm, peak_kind,
                          only=("query_fast",), row_u8=idx.row_u8(), plan=plan, cfg_key=cfg_key)
    query_roof_tc = roofline_tc(prof_query, args.steps, n_loc, nq, idx.row_u8(), peak_bf16())
    step_ms = sum(v[0] for v in prof_query.values()) / args.steps
    step_bytes = 4.0 * d * budget * nq  # candidates_seen x 4d per query
    # bytes the query kernels actually move (ncu dram read + write of the same
    # workload, profiles/ncu_latest.json) over the step's kernel time; the
    # SURVEY 8(d) model (4 d bytes per candidate) is kept beside it: above 1
    # when candidates are verified dataset-major on the tensor cores
    moved, msrc = 0.0, []
    for kq in ("query_fast", "tc_score", "tc_collect", "tc_finish"):
        if kq in prof_query:
            tb, src = ncu_traffic(kq, nq, cfg_key)  # (captured per nq-query batch)
            if tb is None:
                moved = None
                break
            moved += tb
            msrc.append(src)
    query_roof_step = {
        "kernel": "query step (all query kernels)", "bound": "hbm", "unit": "GB/s", "peak": hbm,
        "step_kernel_ms": round(step_ms, 4),
        "dram_bytes": moved,
        "achieved": round(moved / (step_ms / 1e3) / 1e9, 2) if moved else None,
        "frac": round(moved / (step_ms / 1e3) / 1e9 / hbm, 5) if moved else None,
        "dram_source": sorted(set(msrc)) if moved else None,
        "survey_model": {"algorithmic_bytes": step_bytes,
                         "achieved": round(step_bytes / (step_ms / 1e3) / 1e9, 2),
                         "frac": round(step_bytes / (step_ms / 1e3) / 1e9 / hbm, 5),
                         "note": "SURVEY 8(d) bytes (4d per candidate)"}}
    # the reference arm scores its first cpu_queries queries: same subset here
    m_ref = min(args.cpu_queries, nq)
    rec_ref, rat_ref = recall_ratio(out_ids[:m_ref], out_d[:m_ref], out_h[:m_ref], gt_ids[:m_ref],
                                    gt_d[:m_ref], k)
    value = n_total / (build_ms / 1e3) / 1e6
    qps = nq / (query_ms / 1e3)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpoints/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(build_ms, 3),
        "higher_is_better": True, "scaling": args.shard if world > 1 else "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg}: n={n_total}, d={d}, nq={nq}, K=16, L=4, N_r=256, leaf=128, "
                               f"k={k}, c=1.5, beta={args.beta}",
                   "points_per_gpu": n_loc,
                   "sample_mode": args.sample, "parallelism": f"point-shard x{world}",
                   "l2": f"inputs larger than L2 (dataset {n_loc * d * 4 / 1e9:.2f} GB)"},
        "query": {"value": round(qps, 2), "unit": "queries/s", "ms_per_step": round(query_ms, 3),
                  "recall": round(rec, 6), "ratio": round(rat, 6),
                  "recall_on_reference_sample": round(rec_ref, 6),
                  "ratio_on_reference_sample": round(rat_ref, 6), "gpu_launches": query_launches,
                  "roofline": query_roof, "roofline_tc": query_roof_tc, "roofline_step": query_roof_step,
                  "e2e": {"value": round(nq / (e2e_query_ms / 1e3), 2), "unit": "queries/s",
                          "h2d_bytes_per_step": int(nq * d * 4),
                          "d2h_bytes_per_step": int(nq * k * 12 + nq * 20)}},
        "e2e": ({"value": round(n_total / (e2e_build_ms / 1e3) / 1e6, 3), "unit": "Mpoints/s",
                 "h2d_bytes_per_step": int(n_loc * d * 4), "d2h_bytes_per_step": 96} if e2e_build_ms else
                {"value": None, "unit": "Mpoints/s", "note": "c5: the dataset is generated on the device "
                 "(51 GB); the host-buffer build is not timed"}),
        "gpu_launches": build_launches,
        "build_other_sample": {"sample_mode": other, "value": round(n_total / (other_ms / 1e3) / 1e6, 3),
                               "unit": "Mpoints/s", "ms_per_step": round(other_ms, 3),
                               "parity": "hybrid oracle (reference stage functions, same table)"
                               if other == "gpu" else "bit-exact vs reference"},
        "roofline": build_roof,
        "roofline_projection": build_roof_proj,
        "roofline_build_other": build_roof_other,
        "build_stages_ms": {k2: round(v, 3) for k2, v in stage_ms.items()},
        "build_other_stages_ms": {k2: round(v, 3) for k2, v in other_stages.items()},
        "kernels_ms_per_step": {"build": {k2: round(v[0] / args.steps, 4) for k2, v in prof_build.items()},
                                "query": {k2: round(v[0] / args.steps, 4) for k2, v in prof_query.items()}},
        "clocks": clk,
    }
    if devgen:
        line["query"]["recall_queries"] = int(min(nq, args.gt_queries))
    if not args.no_cpu_baseline and world == 1:
        try:
            if devgen:  # the reference on a bounded host copy: the first cpu_build_rows rows
                rows = args.cpu_build_rows or 1_000_000
                base = base_d[:rows].cpu().numpy()
            line["cpu_baseline"] = cpu_baseline(args, base, Q)
            if devgen:
                line["cpu_baseline"]["sample"] = (f"c5 shard: the first {base.shape[0]} of {n} rows (copied to the "
                                                  "host); " + line["cpu_baseline"]["sample"])
        except Exception as e:  # reported, not fatal
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def plumbing(args, rank, world):
    """The multi-rank skeleton of the bench without the GPU work: process group
    (nccl with GPUs, else gloo), the config's point shards, and the all-gather
    of per-shard top-k lists that the query step merges."""
    import torch
    import torch.distributed as dist
    from paper_2406_10938_b200 import data as gen
    from paper_2406_10938_b200.shard import gather_topk, shard_bounds
    backend = "nccl" if torch.cuda.is_available() else "gloo"
    if world > 1:
        dist.init_process_group(backend)
    n = gen.CONFIGS[args.config]["n"]
    s0, s1 = shard_bounds(n, world, rank) if args.shard == "strong" else (rank * n, (rank + 1) * n)
    k, nq = 4, 3
    dev = "cuda" if backend == "nccl" else "cpu"
    # each rank's fake top-k: distances rank + j, ids at the shard's first rows
    d = torch.tensor([[rank + j for j in range(k)]] * nq, dtype=torch.float64, device=dev)
    i = torch.tensor([[s0 + j for j in range(k)]] * nq, dtype=torch.int64, device=dev)
    h = torch.full((nq,), k, dtype=torch.int32, device=dev)
    gd = torch.zeros((world, nq, k), dtype=torch.float64, device=dev)
    gi = torch.zeros((world, nq, k), dtype=torch.int64, device=dev)
    gh = torch.zeros((world, nq), dtype=torch.int32, device=dev)
    if world > 1:
        gather_topk(d, i, h, gd, gi, gh)
        bounds = [None] * world
        dist.all_gather_object(bounds, (s0, s1))
    else:
        gd[0], gi[0], gh[0] = d, i, h
        bounds = [(s0, s1)]
    if rank == 0:
        print(json.dumps({"plumbing": True, "n_gpus": world, "backend": backend, "shard": args.shard,
                          "scaling": args.shard if world > 1 else "weak", "config": args.config,
                          "shards": bounds, "gathered_ids": gi[:, 0, 0].tolist()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def profiled_steps(lib, fn, steps):
    """Per-kernel CUDA-event profile over `steps` extra (untimed) steps; the
    index returned by a build step is dropped right away."""
    import torch
    collect_profile(lib)
    lib.detlsh_profile_enable(1)
    for _ in range(steps):
        out = fn()
        del out
    torch.cuda.synchronize()
    lib.detlsh_profile_enable(0)
    return collect_profile(lib)


def collect_profile(lib):
    import ctypes as C
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data),
                                   C.c_void_p(cnt.ctypes.data), 64)
    keys = names.value.decode().split(";") if m else []
    return {kk: (float(ms[i]), int(cnt[i])) for i, kk in enumerate(keys)}


def roofline_tc(prof, steps, n, nq, row_u8, peak_bf16):
    """tcgen05 scorer: every (row, query) dot product, 2 * R int8 ops each, on the
    tensor pipe.  Peak: dense int8 = 2x dense bf16 on sm_100, so 2x the measured
    bf16 burst figure (MEASURED_PEAKS.json)."""
    if "tc_score" not in prof or not row_u8:
        return None
    ms, launches = prof["tc_score"]
    per_launch_ms = ms / max(1, launches)
    ops = 2.0 * row_u8 * n * nq / max(1, launches / steps)
    ach = ops / (per_launch_ms / 1e3) / 1e12
    op = own_peaks() or {}
    peak = float(op.get("int8_tcgen05_tops", 2.0 * peak_bf16))
    return {"kernel": "tc_score", "bound": "tensor", "unit": "TOPS", "achieved": round(ach, 2),
            "peak": round(peak, 1), "peak_kind": ("measured tcgen05 kind::i8 (profiles/peaks_measured.json)"
                                                  if "int8_tcgen05_tops" in op else "2x measured bf16 burst (dense int8)"),
            "frac": round(ach / peak, 5), "launch_ms": round(per_launch_ms, 4), "int8_ops": ops}


def roofline(prof, steps, n, d, nq, budget, K, L, hbm, peak_kind, only=None, exclude=(),
             row_u8=0, plan=None, cfg_key=None):
    items = [(kk, v) for kk, v in prof.items() if (only is None or kk in only) and kk not in exclude]
    if not items:
        return None
    kern, (ms, launches) = max(items, key=lambda kv: kv[1][0])
    per_launch_ms = ms / max(1, launches)
    if kern == "query_fast" and "tc_score" not in prof:
        plan = None  # no tensor-core hand-off in this run: the kernel verified everything
    b = algo_bytes(kern, n, d, nq, budget, K, L, row_u8, plan)
    total = sum(v[0] for kk, v in prof.items())
    units = nq if kern == "query_fast" else n
    traffic, tsrc = ncu_traffic(kern, units, cfg_key)
    out = {"kernel": kern, "bound": "hbm", "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
           "launch_ms": round(per_launch_ms, 4), "launches_per_step": launches / steps,
           "share_of_kernel_time": round(ms / total, 4) if total else None,
           "traffic": traffic, "traffic_source": tsrc}
    if kern == "project_exact":
        # non-integral data: d x (L K) fp64 FMA chain per point on the FP64
        # tensor pipe (DMMA); peak = tools/probes/peaks.cu's measured DMMA rate
        fl = 2.0 * n * K * L * d
        ach = fl / (per_launch_ms / 1e3) / 1e12
        b = algo_bytes(kern, n, d, nq, budget, K, L)
        op = own_peaks() or {}
        pk = float(op.get("fp64_dmma_tflops", 45.0))
        out.update({"bound": "tensor", "unit": "TFLOP/s", "peak": pk,
                    "peak_kind": ("measured (profiles/peaks_measured.json, tools/probes/peaks.cu)"
                                  if "fp64_dmma_tflops" in op else "nominal B200 FP64 tensor"),
                    "achieved": round(ach, 3), "frac": round(ach / pk, 5), "algorithmic_flops": fl,
                    "hbm_view": {"algorithmic_bytes": b,
                                 "achieved_gbs": round(b / (per_launch_ms / 1e3) / 1e9, 2),
                                 "frac": round(b / (per_launch_ms / 1e3) / 1e9 / hbm, 5)}})
        return out
    if b is None:
        out.update({"achieved": None, "frac": None})
    else:
        ach = b / (per_launch_ms / 1e3) / 1e9
        out.update({"achieved": round(ach, 2), "frac": round(ach / hbm, 5),
                    "algorithmic_bytes": b})
        if kern == "project_tc" and "project_fixup" in prof:
            # the projection stage = the tensor-core pass + its fixup / guarded
            # FP64 pass (both every launch): the same bytes over both
            fx_ms = prof["project_fixup"][0] / max(1, prof["project_fixup"][1])
            sa = b / ((per_launch_ms + fx_ms) / 1e3) / 1e9
            out["stage_with_fixup"] = {"ms": round(per_launch_ms + fx_ms, 4), "achieved": round(sa, 2),
                                       "frac": round(sa / hbm, 5)}
        if plan is not None:
            out["model"] = "plan kernel (tc hand-off): 12 B/leaf x tree-0 leaves + R x tau_rows + n/8 (row bitmap) per query"
        if kern == "query_fast" and row_u8 and plan is None:
            b8 = float(row_u8) * budget * nq  # bytes the u8 rows actually hold
            out["u8_rows"] = {"bytes": b8, "achieved": round(b8 / (per_launch_ms / 1e3) / 1e9, 2),
                              "frac": round(b8 / (per_launch_ms / 1e3) / 1e9 / hbm, 5)}
    return out


if __name__ == "__main__":
    main()
