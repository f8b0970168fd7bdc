"""The C++ drop-in header (include/fastped_b200/fastped.hpp) compiles against the C ABI and, on a
GPU, reproduces the restatement's trajectory (pinned to the reference) step by step."""
import os
import subprocess

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "cpp_api_check.cpp")
LIBDIR = os.path.join(ROOT, "paper_0911_2900_b200")


def build(tmp_path):
    exe = str(tmp_path / "cpp_api_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), SRC,
                    "-L", LIBDIR, "-lfastped_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_header_compiles_and_links(tmp_path):
    assert os.path.exists(build(tmp_path))


def scenario():
    W, H = 40, 30
    c = np.zeros((H, W), np.uint8)
    c[0, :] = c[-1, :] = 1
    c[:, 0] = c[:, -1] = 1
    c[12:18, -1] = 2
    c[5:25, 20] = 1
    c[10, 20] = c[20, 20] = 0
    return c


@pytest.mark.gpu
def test_cpp_drop_in_matches_restatement(tmp_path):
    out = subprocess.run([build(tmp_path), "200"], check=True, capture_output=True, text=True).stdout.splitlines()
    assert out[0] == "errors 3"
    assert out[1] == "blocksize 12500 32767"
    cells = scenario()
    field = O.static_field(cells, 0)
    assert float(out[2].split()[1]) == field[1, 1]
    x, y = O.spawn_agents(cells, 200, 7)
    st = O.State(cells, field, np.asarray(x, np.int32), np.asarray(y, np.int32), 4)
    for s, line in enumerate(out[3:]):
        ex, disp = st.step_once(1.2, 7)
        f = line.split()
        assert int(f[1]) == st.step and int(f[3]) == st.alive_count, line
        assert int(f[5]) == len(ex) and int(f[7]) == disp, line
        assert int(f[9]) == st.hash(), line
    assert len(out) == 3 + 20
