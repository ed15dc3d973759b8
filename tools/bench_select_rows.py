import ctypes as C, time, numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2406_10938_b200 import _lib
lib = _lib.load()
g = np.random.default_rng(1)
rows = [g.normal(size=100000).astype(np.float32) for _ in range(16)]
out = np.zeros(257, np.float32); nd = C.c_uint64(0)
t0 = time.perf_counter()
for r in rows:
    a = r.copy()
    lib.detlsh_select_row_breakpoints(C.c_void_p(a.ctypes.data), 100000, 256, 12345, C.c_void_p(out.ctypes.data), C.byref(nd))
t1 = time.perf_counter()
print(f"{(t1-t0)/16*1e3:.3f} ms per row, draws {nd.value/16:.0f}")
