"""Plan-kernel occupancy A/B (DETLSH_FAST_MINB=3 vs 5) on a config subset."""
import os, sys, time, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg, n, nq = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
if len(sys.argv) > 4:
    import paper_2406_10938_b200 as D
    from paper_2406_10938_b200 import data as gen
    base, Q = gen.make(cfg, n=n, nq=nq)
    idx = D.build_index(base, D.LshParams(beta=0.1, k=50), seed=2)
    for tc in (True, False):
        D.ck_ann_batch(idx, Q, 50, tensor_cores=tc)
        t0 = time.perf_counter()
        for _ in range(3):
            D.ck_ann_batch(idx, Q, 50, tensor_cores=tc)
        dt = (time.perf_counter() - t0) / 3
        print(f"  MINB={os.environ.get('DETLSH_FAST_MINB')} tc={tc}: {dt * 1e3:.1f} ms/batch {nq / dt:.0f} q/s", flush=True)
else:
    for m in ("3", "5"):
        subprocess.run([sys.executable, __file__, cfg, str(n), str(nq), "run"], env=dict(os.environ, DETLSH_FAST_MINB=m))
