"""Standalone DE-Tree build time from device codes (one space), C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, _ = gen.make("c2", nq=16)
idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=2, sample="gpu")
codes = idx.codes()[0]
for rep in range(4):
    t0 = time.perf_counter()
    t = D.build_tree(codes, 0, 128)
    t1 = time.perf_counter()
    print(f"build_tree (host codes, incl. H2D + export-free): {1e3*(t1-t0):.3f} ms")
