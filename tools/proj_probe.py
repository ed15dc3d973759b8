"""Times the exact projection of a config's dataset through the stage function
(detlsh_gpu_project), per profile scope; DETLSH_PROJ_TC=0 forces the FP64 DMMA
kernel.  Usage: python tools/proj_probe.py [config] [n] [reps]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else None
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    import torch
    base, _ = gen.make(cfg, n=n, nq=0)
    n, d = base.shape
    fam = D.sample_hash_family(d, 16, 4, 7)
    X = torch.from_numpy(base).cuda()
    out = torch.empty((4, n, 16), dtype=torch.float32, device="cuda")
    lib = D.load()
    F = torch.from_numpy(np.ascontiguousarray(fam, np.float32)).cuda()
    for r in range(reps + 1):
        if r == 1:
            lib.detlsh_profile_enable(1)
        D._lib.check(lib.detlsh_gpu_project(C.c_void_p(F.data_ptr()), 16, 4, C.c_void_p(X.data_ptr()), n, d,
                                            C.c_void_p(out.data_ptr()), 0, D._lib.F_DEVICE_PTRS))
    torch.cuda.synchronize()
    lib.detlsh_profile_enable(0)
    names = C.create_string_buffer(4096)
    ms = np.zeros(64, np.float64)
    cnt = np.zeros(64, np.uint64)
    m = lib.detlsh_profile_collect(names, 4096, C.c_void_p(ms.ctypes.data), C.c_void_p(cnt.ctypes.data), 64)
    for i, k in enumerate(names.value.decode().split(";")[:m]):
        per = ms[i] / max(1, cnt[i])
        print(f"{k:16s} {per:8.4f} ms/launch  {4.0 * n * d / (per / 1e3) / 1e9:8.1f} GB/s on 4dn  x{cnt[i]}")


if __name__ == "__main__":
    main()
