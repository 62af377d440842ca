"""A small solve with the TMA pair (both geometries, fused closing sweep + residual) and the
TMA SpMV forced on, for compute-sanitizer (memcheck / racecheck) runs."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402
build.build()
from paper_math_9809043_b200.mss import Solver  # noqa: E402
from workloads import make_workload  # noqa: E402

os.environ["MSS_PAIR"] = "1"
for ty in ("16", "8"):
    os.environ["MSS_PAIR_TY"] = ty
    w = make_workload("C2", n=32)
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth)
    x, rep = s.solve(torch.from_numpy(w.f.ravel()).cuda(), rel_tol=w.rel_tol)
    torch.cuda.synchronize()
    print("ty", ty, rep.iters, f"{rep.true_rel_res:.2e}", flush=True)
    s.close()
