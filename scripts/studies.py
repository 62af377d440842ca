"""NEXT-4 studies on the GPU (§Accuracy P:706-737 and the variance
study P:739-755), all through the library's C ABI:

  * base case: power-law log-normal K, variance 2, zero mean, cutoff lengths
    0.016 and 0.002 of the domain oriented at 15 degrees, pressure 1 | 0 on the x-faces,
    no flow on the others — on a 1024^2 grid (the paper's 1000^2 rounded to an integer
    coarsening chain, s = 4);
  * E9 accuracy: x~ = a loose solve (rel 1e-3) of the base case; the manufactured source
    f' = (A x~ - b_0)/V has x~ as its exact discrete solution; solve f' at
    tolerances 1e-1 .. 1e-14 and record fine iterations, RMS and max error against x~, and
    the fitted error reduction per fine iteration (the paper reports ~11);
  * E10 variance: the base field's log rescaled to variances 0.5 .. 6; fine iterations at
    the paper's tolerance (mean-square residual reduced 1e10, i.e. rel 1e-5) and at 1e-10;
  * the same two studies on a 3-D 128^3 power-law field.

Writes profiles/<tag>_studies.json.  usage: python scripts/studies.py [--tag r01]
"""
import argparse
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402

build.build()
from paper_math_9809043_b200.mss import Solver, generate_field  # noqa: E402
from workloads.configs import DIRICHLET, bc_table  # noqa: E402


def fit_reduction(rows):
    """error reduction per fine iteration: slope of log10(rms error) vs fine iterations over
    the rows before the error reaches its floor (round-off)."""
    pts = [(r["iters"][0], r["rms_err"]) for r in rows if r["rms_err"] > 0]
    floor = min(e for _, e in pts)
    use = [(i, e) for i, e in pts if e > 100 * floor]
    if len(use) < 2:
        return None
    it = np.array([p[0] for p in use], dtype=float)
    le = np.log10([p[1] for p in use])
    slope = np.polyfit(it, le, 1)[0]
    return float(10 ** (-slope))


def run_case(ndim, n, ell, theta, log_var_base, variances, tag):
    dev = torch.device("cuda", 0)
    bc = bc_table(ndim, {"x-": (DIRICHLET, 1.0), "x+": (DIRICHLET, 0.0)})
    N = int(np.prod([n[d] for d in range(ndim)]))
    out = {"ndim": ndim, "n": list(n[:ndim]), "model": "power law (1 + r'Lr)^(-1/4)", "ell_cells": list(ell[:ndim]),
           "theta_deg": math.degrees(theta), "log_var": log_var_base}
    t0 = time.perf_counter()
    K = generate_field(ndim, n, 1, ell, theta, 0.0, log_var_base, seed=1998, device=dev)
    torch.cuda.synchronize()
    out["field_ms"] = 1e3 * (time.perf_counter() - t0)
    out["K_ratio"] = float(K.max() / K.min())
    lk = torch.log(K)
    out["log_K_range"] = [float(lk.min()), float(lk.max())]
    s = Solver(ndim, n, K, bc)
    zero = torch.zeros(N, dtype=torch.float64, device=dev)
    x5, r5 = s.solve(zero, rel_tol=1e-5)
    out["base_iters_rel1e-5"] = list(r5.iters)
    # E9
    xt, rt = s.solve(zero, rel_tol=1e-3)
    xt = xt.clone()
    f = s.manufacture_rhs(xt)
    rows = []
    for e in range(1, 15):
        tol = 10.0 ** (-e)
        x, rep = s.solve(f, rel_tol=tol)
        err = x - xt
        rows.append({"rel_tol": tol, "iters": list(rep.iters), "true_rel_res": rep.true_rel_res,
                     "rms_err": float(torch.sqrt(torch.mean(err * err))), "max_err": float(err.abs().max())})
    out["accuracy"] = rows
    out["error_reduction_per_fine_iteration"] = fit_reduction(rows)
    ratios = [r["max_err"] / r["rms_err"] for r in rows if r["rms_err"] > 1e-13]
    out["max_over_rms_error"] = [min(ratios), max(ratios)] if ratios else None
    # E10
    vrows = []
    for v in variances:
        Kv = generate_field(ndim, n, 1, ell, theta, 0.0, v, seed=1998, device=dev)
        sv = Solver(ndim, n, Kv, bc)
        row = {"log_var": v, "K_ratio": float(Kv.max() / Kv.min())}
        for tol in (1e-5, 1e-10):
            x, rep = sv.solve(zero, rel_tol=tol)
            row[f"iters_rel{tol:g}"] = list(rep.iters)
        vrows.append(row)
        del sv, Kv
    out["variance"] = vrows
    print(json.dumps({k: out[k] for k in ("ndim", "n", "K_ratio", "base_iters_rel1e-5",
                                            "error_reduction_per_fine_iteration", "max_over_rms_error")}), flush=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--n2", type=int, default=1024)
    ap.add_argument("--n3", type=int, default=128)
    args = ap.parse_args()
    th = math.radians(15.0)
    n2 = args.n2
    res = {"paper": "accuracy P:706-737 (~11x per iteration, max error within 3x RMS), variance P:739-755 "
                    "(iterations almost constant; variance 3 gives K ratio 8e9)"}
    res["2d"] = run_case(2, (n2, n2, 1), (0.016 * n2, 0.002 * n2), th, 2.0, [0.5, 1.0, 2.0, 3.0, 4.0, 5.0, 6.0], args.tag)
    n3 = args.n3
    res["3d"] = run_case(3, (n3, n3, n3), (0.064 * n3, 0.016 * n3, 0.016 * n3), th, 2.0, [0.5, 1.0, 2.0, 3.0, 4.0],
                         args.tag)
    path = os.path.join(ROOT, "profiles", f"{args.tag}_studies.json")
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
