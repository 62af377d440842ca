"""Setup time (separately from the solve) for the BASELINE configs and for a chain
whose coarsest level sits at the dense-solver cap (N_L = 8192): mss_info's setup_ms and
setup_coarsest_ms (assembly + blocked Cholesky + inverse), after the CUDA module is loaded."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_math_9809043_b200.mss import Solver  # noqa: E402
from workloads import make_workload  # noqa: E402

CASES = [("C2", None, {}), ("C4", None, {}), ("C5", None, {}),
         ("C4", None, {"level_dims": [[128, 128, 128], [64, 64, 128], [16, 16, 32]]})]
w0 = make_workload("C2", n=16)
Solver(w0.ndim, w0.n, torch.from_numpy(w0.K).cuda(), w0.bc, depth=w0.depth).close()   # module load
for name, n, prm in CASES:
    w = make_workload(name, n=n)
    K = torch.from_numpy(w.K).cuda()
    f = torch.from_numpy(w.f.ravel()).cuda()
    for rep in range(2):
        s = Solver(w.ndim, w.n, K, w.bc, depth=None if prm else w.depth, params=prm)
        info = s.info()
        x, r = s.solve(f, rel_tol=w.rel_tol)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, r = s.solve(f, x, rel_tol=w.rel_tol)
        e1.record()
        torch.cuda.synchronize()
        if rep == 1:
            print(f"{name} {w.n} chain {r.dims}: setup {info.setup_ms:.2f} ms (coarsest N_L = "
                  f"{r.dims[-1][0] * r.dims[-1][1] * r.dims[-1][2]}: {info.setup_coarsest_ms:.2f} ms), "
                  f"solve {e0.elapsed_time(e1):.2f} ms, iters {r.iters}")
        s.close()
