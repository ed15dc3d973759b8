"""Does in-process NVML clock polling (bench.py's ClockSampler) slow builds down?
Times back-to-back GPU-sample and reference-sample builds with and without a 100 ms
NVML poller thread."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import pynvml
import paper_2406_10938_b200 as D
from paper_2406_10938_b200 import data as gen
base, _ = gen.make("c2", nq=16)
dev = torch.from_numpy(base).cuda()
p = D.LshParams(beta=0.1, k=50)
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False
lat = []


def poll():
    while not stop:
        t0 = time.perf_counter()
        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        lat.append(time.perf_counter() - t0)
        time.sleep(0.1)


def run(mode, reps=10):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = D.build_index(dev, p, seed=2, sample=mode, borrow=True, keep_codes=False)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return " ".join(f"{t:.1f}" for t in ts)


for mode in ("gpu", "reference"):
    run(mode, 3)
    print(mode, "no poller :", run(mode))
    stop = False
    th = threading.Thread(target=poll, daemon=True)
    th.start()
    print(mode, "NVML 100ms:", run(mode))
    stop = True
    th.join()
print("NVML poll latency ms: max %.2f mean %.2f" % (max(lat) * 1e3, sum(lat) / len(lat) * 1e3))
