"""Feasibility probe: do two independent C5 solves on two streams overlap one solve's
latency-bound coarse phases (level 1, cluster tail) with the other's HBM-bound level 0?
Two full contexts (separate operators), two host threads.  Prints the single-solve time and
the time for both solves launched together."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_math_9809043_b200.mss import Solver
from workloads import make_workload

case = (sys.argv[1] if len(sys.argv) > 1 else "C5", int(sys.argv[2]) if len(sys.argv) > 2 else None)
NCTX = int(os.environ.get("NCTX", "2"))
w = make_workload(*case)
K = torch.from_numpy(w.K).cuda()
f = torch.from_numpy(np.ascontiguousarray(w.f, dtype=np.float64).ravel()).cuda()
pri = [int(p) for p in os.environ.get("PRIO", "0,0,0,0").split(",")]
ctx = []
for i in range(NCTX):
    st = torch.cuda.Stream(priority=pri[i])
    with torch.cuda.stream(st):
        s = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, stream=st)
    ctx.append((s, st, torch.empty_like(f)))
torch.cuda.synchronize()

def one(i, reps, out):
    s, st, x = ctx[i]
    with torch.cuda.stream(st):
        for _ in range(reps):
            _, rep = s.solve(f, x=x, rel_tol=w.rel_tol)
        st.synchronize()
    out[i] = list(rep.iters)

out = [None] * NCTX
for i in range(NCTX):
    one(i, 2, out)
torch.cuda.synchronize()
t0 = time.perf_counter(); one(0, 4, out); t1 = time.perf_counter()
print(f"single: {(t1 - t0) / 4 * 1e3:.2f} ms per solve, iters {out[0]}")
for reps in (4, 8):
    th = [threading.Thread(target=one, args=(i, reps, out)) for i in range(NCTX)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for t in th: t.start()
    for t in th: t.join()
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    dt = (t1 - t0) / reps
    print(f"{NCTX} concurrent x{reps}: {dt * 1e3:.2f} ms per round of {NCTX} solves = {dt / NCTX * 1e3:.2f} ms per solve, "
          f"{NCTX * w.N / dt:.3e} unknowns/s, iters {out}")
