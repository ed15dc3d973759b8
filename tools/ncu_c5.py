"""C5 (1e8 x 128, generated on the device): GPU-sample build + one query batch,
for an ncu capture of tc_score / query_fast at full scale.  Usage: python tools/ncu_c5.py [nq]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_10938_b200 as D  # noqa: E402
from paper_2406_10938_b200 import data as gen  # noqa: E402

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
base, Q = gen.make_device("c5", nq=nq)
idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=5, sample="gpu", borrow=True, keep_codes=False)
k = 50
ids = torch.empty((nq, k), dtype=torch.int32, device="cuda")
ds = torch.empty((nq, k), dtype=torch.float64, device="cuda")
D.ck_ann_device(idx, Q, k, ids, ds)
torch.cuda.synchronize()
print("done c5", nq)
