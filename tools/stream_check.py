"""Checks that a device-mode query batch is ordered on the caller's stream:
CUDA events on that stream must bracket its kernels."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

base, Q = gen.make("c2")
X = torch.from_numpy(base).cuda()
idx = D.build_index(X, D.LshParams(beta=0.1, k=50), seed=2, borrow=True, keep_codes=False)
Qd = torch.from_numpy(Q).cuda()
nq, k = Q.shape[0], 50
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
ds = torch.empty((nq, k), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
for prof in (0, 1):
    D.load().detlsh_profile_enable(prof)
    for _ in range(2):
        D.ck_ann_device(idx, Qd, k, ids, ds, stream=st.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(st)
    for _ in range(3):
        D.ck_ann_device(idx, Qd, k, ids, ds, stream=st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"profile={prof}: events {e0.elapsed_time(e1) / 3:.3f} ms/batch, wall {1e3 * (t1 - t0) / 3:.3f} ms/batch")
