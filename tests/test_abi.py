"""CPU-only checks of the C ABI: the library builds for sm_100a, loads, and exports
every function include/mss.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mss.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s+\*?(mss_[A-Za-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_math_9809043_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ["mss_setup", "mss_solve", "mss_free", "mss_solve_host", "mss_solve_host_batch", "mss_apply_A", "mss_smooth",
                 "mss_residual_restrict", "mss_prolong_add", "mss_precond", "mss_coarse_solve",
                 "mss_dot", "mss_get_faces", "mss_setup_dist", "mss_nccl_unique_id"]:
        assert must in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_covers_header(lib_path):
    from paper_math_9809043_b200 import mss
    bound = {n for n, _, _ in mss.SIGNATURES}
    assert set(declared_functions()) <= bound
    lib = mss.load_library()
    p = mss.default_params()
    assert (p.scale, p.m, p.f, p.interp, p.use_lift) == (4, 4, 0.1, 0, 1)
    assert lib.mss_strerror(-6).decode() == "PCG breakdown"


def test_sass_is_sm100a(lib_path):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib_path], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_slab_range_partitions(lib_path):
    from paper_math_9809043_b200 import mss
    lib = mss.load_library()
    n = (ctypes.c_int64 * 3)(512, 512, 512)
    ends = []
    for r in range(8):
        zb, ze = ctypes.c_int64(), ctypes.c_int64()
        assert lib.mss_slab_range(n, 3, None, -1, r, 8, ctypes.byref(zb), ctypes.byref(ze)) == 0
        ends.append((zb.value, ze.value))
    assert ends[0][0] == 0 and ends[-1][1] == 512
    assert all(ends[i][1] == ends[i + 1][0] for i in range(7))
