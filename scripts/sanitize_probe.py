"""Small solves exercising every kernel family (grid, column-walk, both cluster tails,
comparison methods, loopback slabs) for compute-sanitizer runs."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_math_9809043_b200 import build  # noqa: E402
build.build()
from paper_math_9809043_b200.mss import Solver, LoopbackGroup, slab_range  # noqa: E402
from workloads import make_workload  # noqa: E402


def run(w, **params):
    s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, params=params)
    x, rep = s.solve(torch.from_numpy(w.f.ravel()).cuda(), rel_tol=w.rel_tol)
    torch.cuda.synchronize()
    print(w.name, params, rep.iters, rep.tail_kind, f"{rep.true_rel_res:.2e}", flush=True)
    s.close()


run(make_workload("C2", n=64))                              # col-walk + smem tail
run(make_workload("C5", n=128), tail_cells=40000)           # smem tail on 32^3
os.environ["MSS_NO_TAILSM"] = "1"
run(make_workload("C5", n=128))                             # L2-resident cluster tail
del os.environ["MSS_NO_TAILSM"]
run(make_workload("C3", n=256), use_lift=0, interp=1)       # 2-D
run(make_workload("C1"))
run(make_workload("C2", n=32), method=1)
run(make_workload("C2", n=32), method=3)
os.environ["MSS_PAIR"] = "1"
run(make_workload("C2", n=64))
del os.environ["MSS_PAIR"]
# loopback slabs, 2 ranks
w = make_workload("C5", n=64)
grp = LoopbackGroup(2)
prm = {"gather_below": 4096}


def rank(r):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        z0, z1 = slab_range(w.n, r, 2, params=prm)
        s = Solver(w.ndim, w.n, torch.from_numpy(np.ascontiguousarray(w.K[:, z0:z1])).cuda(), w.bc, params=prm,
                   stream=st, comm=("loop", grp, r))
        x, rep = s.solve(torch.from_numpy(np.ascontiguousarray(w.f[z0:z1]).ravel()).cuda())
        st.synchronize()
        print("loopback rank", r, rep.iters, flush=True)
        s.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(2)]
[t.start() for t in th]
[t.join() for t in th]
grp.close()
print("sanitize probe done")
