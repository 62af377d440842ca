"""Run the CPU oracle ONCE on a full BASELINE config (default C5, 512^3) and record its
per-level iteration counts, true residual and a seeded sample of its solution.

Test infrastructure (calls only ``oracle/`` and ``workloads/``): the output
``tests/golden/<cfg>_oracle.json`` is the stored expectation that
``tests/test_gpu_fullsize.py`` compares the GPU solve with at full size (VERDICT r1
"Next" 1: "Run the oracle once on full C5 ... record its per-level counts").
estimates 20-30 GiB of host RAM and tens of minutes for C5.

    python scripts/oracle_c5.py [C5] [--n N]
"""
import argparse
import json
import os
import resource
import sys
import time

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from oracle import mss_oracle as O  # noqa: E402
from workloads import make_workload  # noqa: E402


def sample_cells(shape, n=4096, seed=11):
    """Seeded flat indices (x fastest) plus the domain's corners and face centres."""
    rng = np.random.default_rng(seed)
    N = int(np.prod(shape))
    idx = set(int(v) for v in rng.integers(0, N, size=n))
    nz, ny, nx = shape
    for k in (0, nz // 2, nz - 1):
        for j in (0, ny // 2, ny - 1):
            for i in (0, nx // 2, nx - 1):
                idx.add(i + nx * (j + ny * k))
    return sorted(idx)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg", nargs="?", default="C5")
    ap.add_argument("--n", type=int, default=None, help="reduced size (same recipe)")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    t0 = time.perf_counter()
    w = make_workload(a.cfg, a.n)
    t1 = time.perf_counter()
    o = O.MultiScaleOracle(w.ndim, w.n, w.K, w.bc, depth=w.depth)
    t2 = time.perf_counter()
    x, info = o.solve(w.f, w.rel_tol)
    t3 = time.perf_counter()
    idx = sample_cells(w.shape)
    xf = x.ravel()
    rec = {
        "cfg": a.cfg,
        "n": list(w.n),
        "note": w.note,
        "levels": [list(d) for d in o.dims],
        "iters": [int(v) for v in info.iters],
        "calls": [int(v) for v in info.calls],
        "not_converged": bool(info.not_converged),
        "true_rel_res": info.true_rel_res,
        "min_margin": info.min_margin,
        "x_l2": float(np.linalg.norm(xf)),
        "x_sum": float(xf.sum()),
        "sample_idx": idx,
        "sample_x": [float(xf[i]) for i in idx],
        "seconds": {"workload": t1 - t0, "setup": t2 - t1, "solve": t3 - t2},
        "peak_rss_gib": resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20,
        "host": {"cpus": os.cpu_count(), "threads_used": 1},
        "script": "scripts/oracle_c5.py (oracle/ + workloads/ only)",
    }
    tag = a.cfg.lower() + (f"_{a.n}" if a.n else "")
    out = a.out or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden",
                                f"{tag}_oracle.json")
    with open(out, "w") as fh:
        json.dump(rec, fh)
    print(json.dumps({k: v for k, v in rec.items() if not k.startswith("sample")}))


if __name__ == "__main__":
    main()
