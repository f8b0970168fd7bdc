"""The device weight function restates glibc 2.39's exp (paper_0911_2900_b200/csrc/fp_exp.h).
Compiled for the host here and compared bit-for-bit with this machine's libm `exp` -- the
function the reference calls (planning.hpp:102).  CPU only."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def lib():
    d = tempfile.mkdtemp()
    so = os.path.join(d, "exp_check.so")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", so,
                    os.path.join(HERE, "native", "exp_check.c"), "-lm"], check=True)
    L = C.CDLL(so)
    L.compare_range.restype = C.c_int64
    L.compare_range.argtypes = [C.c_double, C.c_double, C.c_int64, C.c_uint64, C.POINTER(C.c_double)]
    L.compare_lattice.restype = C.c_int64
    L.compare_lattice.argtypes = [C.c_double, C.c_int64, C.c_uint64, C.POINTER(C.c_double)]
    L.restated_exp.restype = C.c_double
    L.restated_exp.argtypes = [C.c_double]
    return L


@pytest.mark.parametrize("lo,hi", [(-12, 12), (-1e-3, 1e-3), (-700, 700), (-745.2, -700), (700, 709.8),
                                   (-1100, 1100), (-1e-17, 1e-17), (-60, 60)])
def test_range_bitwise(lib, lo, hi):
    bad = C.c_double()
    assert lib.compare_range(lo, hi, 1_500_000, 7, C.byref(bad)) == 0, bad.value


@pytest.mark.parametrize("k_s", [1.2, 0.5, 3.0, 0.0])
def test_hot_path_lattice_bitwise(lib, k_s):
    bad = C.c_double()
    assert lib.compare_lattice(k_s, 1_000_000, 11, C.byref(bad)) == 0, bad.value


def test_specials(lib):
    import math
    for x in (0.0, -0.0, 1e-300, -1e-300, float("inf"), float("-inf"), 709.78, -708.5, -745.1, 1e5, -1e5):
        want = math.exp(x) if x < 709.8 else float("inf")
        assert lib.restated_exp(x) == want
    assert math.isnan(lib.restated_exp(float("nan")))
