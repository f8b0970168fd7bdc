"""The C ABI library builds for sm_100a, loads, and exports every entry point declared in
include/fastped_b200.h; without a GPU every compute call fails loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fastped_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\*\s]+?)\b(fp_\w+)\s*\(", txt, re.M)))


def test_header_declares_the_surface():
    names = declared()
    for must in ("fp_create", "fp_plan", "fp_move", "fp_step", "fp_run", "fp_get_occupancy",
                 "fp_get_agents", "fp_state_hash", "fp_static_field", "fp_spawn_agents"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_0911_2900_b200 import fastped as fp
    L = fp.library()
    out = subprocess.run(["nm", "-D", "--defined-only", fp.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (fp_\w+)", out))
    for name in declared():
        assert name in exported, name
        assert hasattr(L, name)
    assert set(fp.SIGNATURES) == set(declared())


def test_library_is_sm100a():
    from paper_0911_2900_b200 import fastped as fp
    fp.library()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", fp.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_compute_fails_loudly_without_gpu():
    from paper_0911_2900_b200 import fastped as fp
    if fp.cuda_available():
        pytest.skip("a GPU is present")
    g = fp.from_rows(["#####", "#..E#", "#####"])
    with pytest.raises(fp.DeviceError):
        fp.compute_static_field(g)
    with pytest.raises(fp.DeviceError):
        fp.SimState(g, None, fp.roster([(1, 1)], 1))


def test_host_validation_messages():
    from paper_0911_2900_b200 import fastped as fp
    with pytest.raises(ValueError, match="closed boundary"):
        fp.from_rows(["###", "#..", "###"])
    with pytest.raises(ValueError, match="periodic-x"):
        fp.from_rows(["#.#", "...", "###"], boundary=fp.PERIODIC_X)
    assert fp.compute_blocksize(100000, 8) == 12500
    with pytest.raises(ValueError, match="cores must be >= 1"):
        fp.compute_blocksize(100, 0)
    with pytest.raises(ValueError, match="k_other"):
        fp.SimParams(k_other=0.5).validate()
    with pytest.raises(RuntimeError, match="free cells"):
        fp.spawn_agents(fp.from_rows(["###", "#.#", "###"]), 2, 4, 1)


def test_spawn_matches_oracle():
    import oracle as O
    from paper_0911_2900_b200 import fastped as fp
    from tests.helpers import random_grid
    r = np.random.default_rng(2)
    cells = random_grid(r, 50, 40, 0.2, 2)
    ro = fp.spawn_agents(fp.Grid(cells), 300, 4, 77)
    x, y = O.spawn_agents(cells, 300, 77)
    assert (ro.x == x).all() and (ro.y == y).all()
