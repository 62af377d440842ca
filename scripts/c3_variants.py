"""C3 (2-D 1024^2, layered K with contrast 1e9) timed with and without the lift, as SURVEY
§8(d) asks: with the lift x0 = P_bf is the exact discrete solution (P2-ii), so the solve
takes 0 iterations; without it (x0 = 0) the solver does real work.  Every solve starts from
x = 0 (reset outside the timed events).  Diagnostic; prints one line per variant."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402

build.build()
from paper_math_9809043_b200.mss import MSSError, Solver  # noqa: E402
from workloads import make_workload  # noqa: E402

w = make_workload("C3")
K = torch.from_numpy(w.K).cuda()
f = torch.from_numpy(w.f.ravel()).cuda()
# linear E without the lift stagnates: capped at 20 iterations per call, or
# the recursion multiplies 500-iteration calls
for prm in ({}, {"use_lift": 0, "interp": 1}, {"use_lift": 0, "max_iter": 20}):
    s = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, params=prm)
    x = torch.zeros(s.N, dtype=torch.float64, device="cuda")
    times = []
    try:
        for rep in range(6 if prm.get("max_iter") is None else 2):
            x.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            x, r = s.solve(f, x, rel_tol=w.rel_tol)
            e1.record()
            torch.cuda.synchronize()
            if rep:
                times.append(e0.elapsed_time(e1))
        times.sort()
        ms = times[len(times) // 2]
        print(json.dumps({"params": prm, "iters": list(r.iters), "calls": list(r.calls), "true_rel_res": r.true_rel_res,
                          "rc": r.rc, "ms": ms, "unknowns_per_s": w.N / ms * 1e3}), flush=True)
    except MSSError as e:
        print(json.dumps({"params": prm, "error": str(e)}), flush=True)
    s.close()
