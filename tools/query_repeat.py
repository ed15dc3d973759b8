"""Per-call wall time of repeated device-resident query batches on a config
(looks for per-call host waits: scratch growth, syncs)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
base, Q = gen.make(cfg)
X = torch.from_numpy(base).cuda()
idx = D.build_index(X, D.LshParams(beta=0.1, k=50), seed=2, borrow=True, keep_codes=False)
Qd = torch.from_numpy(Q).cuda()
nq, k = Q.shape[0], 50
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
ds = torch.empty((nq, k), dtype=torch.float64, device="cuda")
lib = D.load()
if os.environ.get("QR_PROFILE"):
    lib.detlsh_profile_enable(1)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.ck_ann_device(idx, Qd, k, ids, ds)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"call {r}: enqueue {1e3 * (t1 - t0):.2f} ms, total {1e3 * (t2 - t0):.2f} ms", flush=True)
