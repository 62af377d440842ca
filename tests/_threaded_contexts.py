"""Helper run by tests/test_gpu_parity.py::test_contexts_on_parallel_host_threads in a fresh
process (so every process-wide host cache starts cold): four contexts of different shapes are
set up and solved concurrently from host threads, each on its own stream (ctypes releases the
GIL, so the C library really runs in parallel), then the same solves run again one by one.
Prints "OK" when every solution and count is bitwise identical."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_math_9809043_b200.mss import Solver  # noqa: E402
from workloads import make_workload  # noqa: E402

CASES = [("C5", 128), ("C2", None), ("C4", 64), ("C3", 256)]


def run(case, out, i):
    w = make_workload(*case)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s = Solver(w.ndim, w.n, torch.from_numpy(w.K).cuda(), w.bc, depth=w.depth, stream=st)
        f = torch.from_numpy(np.ascontiguousarray(w.f, dtype=np.float64).ravel()).cuda()
        x, rep = s.solve(f, rel_tol=w.rel_tol)
        st.synchronize()
        out[i] = (x.cpu().numpy(), list(rep.iters), rep.true_rel_res)
        s.close()


def main():
    par = [None] * len(CASES)
    th = [threading.Thread(target=run, args=(c, par, i)) for i, c in enumerate(CASES)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    seq = [None] * len(CASES)
    for i, c in enumerate(CASES):
        run(c, seq, i)
    for c, a, b in zip(CASES, par, seq):
        assert a is not None, c
        assert a[1] == b[1] and a[2] == b[2], (c, a[1], b[1])
        assert np.array_equal(a[0], b[0]), c
    print("OK", [a[1] for a in par])


if __name__ == "__main__":
    main()
