"""Diagnostic: launch individual level-0 kernels of the C5 512^3 context through the C-ABI
hooks (prolongation, residual + restriction, operator apply), so ncu can capture exactly
those launches (-k regex:<kernel> -c 1).  Prints event timings.  Not a bench line."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402

build.build()
from paper_math_9809043_b200.mss import Solver, generate_field  # noqa: E402

n = (512, 512, 512)
K = generate_field(3, n, 1, (16.0, 16.0, 16.0), 0.0, 0.0, 2.0, seed=4)
bc = [(1, 1.0), (1, 0.0), (0, 0.0), (0, 0.0), (0, 0.0), (0, 0.0)]
s = Solver(3, n, K, bc)
N0, N1 = s.level_N(0), s.level_N(1)
g = torch.Generator(device="cuda").manual_seed(1)
r = torch.randn(N0, dtype=torch.float64, device="cuda", generator=g)
z = torch.randn(N0, dtype=torch.float64, device="cuda", generator=g)
y = torch.randn(N1, dtype=torch.float64, device="cuda", generator=g)
which = sys.argv[1:] or ["prolong", "resid", "apply"]
for w in which:
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if w == "prolong":
            s.prolong_add(0, y, z, 1)
        elif w == "resid":
            s.residual_restrict(0, r, z)
        elif w == "apply":
            s.apply_A(0, z)
        e1.record()
        torch.cuda.synchronize()
        print(w, f"{e0.elapsed_time(e1):.3f} ms (incl. hook copies)")
