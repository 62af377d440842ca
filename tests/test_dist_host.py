"""CPU tests (gloo, world_size 2) of the multi-rank host logic around the z-slab solver:
NCCL-id broadcast over the process group, slab partition from the library, slab slicing
of the seeded inputs, and the max-over-ranks timing reduction used by bench.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_math_9809043_b200 import dist as D
        from paper_math_9809043_b200 import mss
        from workloads import make_workload
        out = {}
        # 1. id broadcast: rank 0's bytes arrive unchanged everywhere
        payload = bytes(range(128)) if rank == 0 else None
        got = D.broadcast_bytes(payload, 128, device="cpu")
        out["id_ok"] = got == bytes(range(128))
        # 2. slab partition of C5's recipe at 128^3 (ndist = 2 with gather_below 32768)
        prm = {"gather_below": 32768}
        zr = mss.slab_range((128, 128, 128), rank, world, params=prm)
        zs = [None] * world
        dist.all_gather_object(zs, zr)
        out["slabs"] = zs
        # 3. the slabs of the seeded inputs tile the full arrays
        w = make_workload("C5", n=32)
        zr32 = mss.slab_range((32, 32, 32), rank, world, params={"gather_below": 512})
        Ks = D.slab_arrays(w.K, zr32)
        parts = [None] * world
        dist.all_gather_object(parts, Ks)
        out["tile_ok"] = bool(np.array_equal(np.concatenate(parts, axis=1), w.K))
        # 4. slowest-rank timing
        out["max"] = D.max_over_ranks(1.0 + rank)
        out["sum"] = D.sum_over_ranks(1.0 + rank)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        o = res[r]
        assert o["id_ok"]
        assert o["slabs"] == [(0, 64), (64, 128)]
        assert o["tile_ok"]
        assert o["max"] == 2.0 and o["sum"] == 3.0


def test_slab_units_and_errors():
    from paper_math_9809043_b200 import mss
    # C5: ndist = 2 (512^3 and 128^3 distributed; 32^3 >= 64^3? no -> replicated), unit 16
    ranges = [mss.slab_range((512, 512, 512), r, 8) for r in range(8)]
    assert ranges == [(64 * r, 64 * (r + 1)) for r in range(8)]
    ranges3 = [mss.slab_range((512, 512, 512), r, 3) for r in range(3)]
    assert ranges3[0][0] == 0 and ranges3[-1][1] == 512
    assert all(a % 16 == 0 and b % 16 == 0 for a, b in ranges3)
    with pytest.raises(mss.MSSError):
        mss.slab_range((512, 512, 512), 0, 64)        # 32 units < 64 ranks
