"""Diagnostic: solve one config a few times and print the per-kernel / per-level timing
breakdown the library measures live (mss_profile).  Not a bench line."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402
from workloads import make_workload  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tail", type=int, default=65536)
ap.add_argument("--prof-level", type=int, default=8)
ap.add_argument("--params", default="{}")
ap.add_argument("--stream", action="store_true", help="run on a non-default stream")
args = ap.parse_args()
build.build()
from paper_math_9809043_b200.mss import Solver, load_library  # noqa: E402

if os.environ.get("MSS_PROBE_LIB"):   # A/B against another build of the library (same session)
    load_library(os.path.join(ROOT, os.environ["MSS_PROBE_LIB"]))

if args.stream:
    torch.cuda.set_stream(torch.cuda.Stream())
w = make_workload(args.config, n=args.n)
K = torch.from_numpy(w.K).cuda()
f = torch.from_numpy(w.f.ravel()).cuda()
prm = {"tail_cells": args.tail, **json.loads(args.params)}
s = Solver(w.ndim, w.n, K, w.bc, depth=w.depth, params=prm)
x, rep = s.solve(f, rel_tol=w.rel_tol)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(args.reps):
    x, rep = s.solve(f, x, rel_tol=w.rel_tol)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / args.reps
print(f"{args.config} n={w.n} levels={rep.dims} iters={rep.iters} calls={rep.calls} res={rep.true_rel_res:.2e} "
      f"tail level {rep.tail_level} kind {rep.tail_kind}")
print(f"  solve {ms:.3f} ms  ->  {w.N / ms * 1e3:.4g} unknowns/s, launches/solve {rep.kernel_launches}")
s.profile(True, args.prof_level)
t0 = time.perf_counter()
x, rep = s.solve(f, x, rel_tol=w.rel_tol)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
prof = s.profile_read()
s.profile(False, 0)
tot = sum(v[1] for v in prof.values())
print(f"  profiled solve wall {wall:.2f} ms, sum of bracketed kernels {tot:.2f} ms")
for (name, lvl), (c, m, by) in sorted(prof.items(), key=lambda kv: -kv[1][1]):
    gbs = by / (m / 1e3) / 1e9 if m > 0 and by > 0 else 0
    print(f"  L{lvl} {name:16s} n={c:6d} ms={m:9.3f} avg_us={1e3 * m / c:9.2f} GB/s={gbs:8.1f}")
