"""Build-stage timings (host-side ms) and per-kernel profile for one config/sample mode."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "gpu"
base, _ = gen.make(cfg, nq=16)
dev = torch.from_numpy(base).cuda()
p = D.LshParams(beta=0.1, k=50)
for _ in range(3):
    idx = D.build_index(dev, p, seed=2, sample=mode, borrow=True, keep_codes=False)
torch.cuda.synchronize()
lib = D.load()
lib.detlsh_profile_enable(1)
t0 = time.perf_counter()
idx = D.build_index(dev, p, seed=2, sample=mode, borrow=True, keep_codes=False)
torch.cuda.synchronize()
t1 = time.perf_counter()
lib.detlsh_profile_enable(0)
print(f"{cfg} {mode}: wall {1e3 * (t1 - t0):.2f} ms")
for k, v in idx.build_timings().items():
    print(f"  stage {k:20s} {v:8.3f} ms")
names = C.create_string_buffer(4096)
ms = np.zeros(64)
cnt = np.zeros(64, np.uint64)
m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
for i, nm in enumerate(names.value.decode().split(";")[:m]):
    print(f"  kernel {nm:20s} {ms[i]:8.3f} ms x{int(cnt[i])}")
