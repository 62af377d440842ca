"""Beyond the BASELINE configs: one solve of the C5 recipe scaled to n^3 (default 1024^3 =
1.07e9 unknowns) on ONE B200, to show the HBM layout holding a billion-cell
problem in 180 GB.  K is generated on the device (mss_field_generate, Gaussian log-normal,
correlation n/32 cells, log-variance 2.2 -> max/min ~1e6 like C5 at 1024^3), so the host never holds
an n^3 array.  Diagnostic, not a bench line; prints one JSON line (profiles/r01j_big.json is that line).

usage: python scripts/big.py [--n 1024] [--tag r01j]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402

build.build()
from paper_math_9809043_b200.mss import Solver, generate_field  # noqa: E402
from workloads.configs import DIRICHLET, bc_table  # noqa: E402


def used_gb():
    free, total = torch.cuda.mem_get_info()
    return (total - free) / 1e9, total / 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tag", default="r01j")
    ap.add_argument("--log-var", type=float, default=2.2)
    args = ap.parse_args()
    n = args.n
    N = n ** 3
    dev = torch.device("cuda", 0)
    out = {"n": [n, n, n], "unknowns": N, "recipe": "C5 scaled: Gaussian log-normal K, correlation n/32 cells, "
           f"log-variance {args.log_var}, p = 1 | 0 on the x-faces, no flow elsewhere, f = 0, rel_tol 1e-10"}
    t0 = time.perf_counter()
    K = generate_field(3, (n, n, n), model=0, ell=(n / 32.0,) * 3, log_var=args.log_var, seed=4, device=dev)
    torch.cuda.synchronize()
    out["field_s"] = time.perf_counter() - t0
    out["K_ratio"] = float(K.max() / K.min())
    bc = bc_table(3, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    t0 = time.perf_counter()
    s = Solver(3, (n, n, n), K, bc)
    torch.cuda.synchronize()
    out["setup_s"] = time.perf_counter() - t0
    del K
    torch.cuda.empty_cache()
    f = torch.zeros(N, dtype=torch.float64, device=dev)
    x = torch.zeros(N, dtype=torch.float64, device=dev)
    x, rep = s.solve(f, x, rel_tol=1e-10)
    torch.cuda.synchronize()
    out["hbm_used_gb"], out["hbm_total_gb"] = used_gb()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        x, rep = s.solve(f, x, rel_tol=1e-10)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    out.update({"levels": rep.dims, "iters_per_level": list(rep.iters), "true_rel_res": rep.true_rel_res,
                "solve_ms": ms, "unknowns_per_s": N / ms * 1e3, "ns_per_unknown": ms * 1e6 / N})
    print(json.dumps(out), flush=True)
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_big.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
