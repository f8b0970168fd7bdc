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


HARNESS = os.path.join(ROOT, "tests", "native", "harness_check.cpp")


def build_harness(tmp_path):
    exe = str(tmp_path / "harness_check")
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), HARNESS,
                    "-L", LIBDIR, "-lfastped_b200", f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_cpp_harness_host_side(tmp_path):
    """The C++ harness header: scenario text round trip and errors, the reference's CSV bytes
    (tests/test_scenario_io.cpp:93-105, test_bench.cpp:78-83,181-184), Weidmann and capacity
    known answers (test_bench.cpp:85-94,162-171)."""
    out = subprocess.run([build_harness(tmp_path), "--host"], check=True, capture_output=True,
                         text=True).stdout.splitlines()
    assert out[0] == "roundtrip 1"
    assert out[1].startswith("error scenario line 1: malformed header")
    assert out[2:4] == ["scenario,agents_initial,v_max,cores,steps,wall_time_s,plan_time_s,move_time_s,seed",
                        "plaza,1000,4,8,396,1.500000,1.250000,0.125000,42"]
    assert out[4:6] == ["scenario,agents_initial,v_max,cores,wall_time_s,factor", "syn,10,4,2,0.500000,1.235"]
    assert out[6:8] == ["density,mean_speed,flow", "0.500000,1.600000,0.800000"]
    w1, w3 = map(float, out[8].split()[1:])
    assert abs(w1 - 1.0580628560768004) < 1e-9 and abs(w3 - 0.330694766470473) < 1e-9
    assert out[9] == "capacity 198000 128000 256000"


@pytest.mark.gpu
def test_cpp_fundamental_diagram_matches_reference(tmp_path):
    out = subprocess.run([build_harness(tmp_path)], check=True, capture_output=True, text=True).stdout.splitlines()
    fd = [tuple(map(float, l.split()[1:])) for l in out if l.startswith("fd ")]
    corridor = np.zeros((5, 25), np.uint8)
    corridor[0, :] = corridor[-1, :] = 1
    d, s, f = O.ref_fundamental_diagram(corridor, 0.4, 4, [0.5, 1.0, 2.0, 4.0], 9, 50, 120)
    assert fd == list(zip(d, s, f))
