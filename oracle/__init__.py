"""ctypes handles on the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle`` -- oracle/liboracle.so, the plain-C restatement of the reference hot path.
* ``Reference`` -- oracle/_ref/libfastped_ref.so, the unmodified reference headers behind an
  extern "C" shim (built only where /root/reference exists; travels to the GPU box prebuilt).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this package.  The product (paper_0911_2900_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfastped_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and oracle/_ref when the reference headers are present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OrcState(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("boundary", C.c_int32),
        ("cells", C.c_void_p), ("field", C.c_void_p), ("n", C.c_int32),
        ("x", C.c_void_p), ("y", C.c_void_p), ("v_max", C.c_void_p), ("alive", C.c_void_p),
        ("occ", C.c_void_p), ("desired_x", C.c_void_p), ("desired_y", C.c_void_p),
        ("step", C.c_int64), ("alive_count", C.c_int64), ("potential", C.c_int32),
        ("drive_gradient", C.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_rng_u64.restype = C.c_uint64
        L.orc_rng_u64.argtypes = [C.c_uint64] * 4
        L.orc_unit_interval.restype = C.c_double
        L.orc_unit_interval.argtypes = [C.c_uint64]
        L.orc_compute_blocksize.restype = C.c_int
        L.orc_compute_blocksize.argtypes = [C.c_int64, C.c_int]
        L.orc_static_field.argtypes = [C.c_int32, C.c_int32, C.c_int32, _u8p, _f64p]
        L.orc_enumerate_candidates.restype = C.c_int
        L.orc_enumerate_candidates.argtypes = [C.POINTER(OrcState), C.c_int32, _i32p, _i32p]
        L.orc_sample_index.restype = C.c_int64
        L.orc_sample_index.argtypes = [_f64p, C.c_int64, C.c_double]
        L.orc_choice_weights.restype = C.c_int
        L.orc_choice_weights.argtypes = [C.POINTER(OrcState), C.c_int32, C.c_double, _f64p, _i32p, _i32p]
        L.orc_plan_phase.argtypes = [C.POINTER(OrcState), C.c_double, C.c_uint64]
        L.orc_movement_order.argtypes = [C.c_int64, C.c_uint64, C.c_int64, _u32p]
        L.orc_move_phase.restype = C.c_int64
        L.orc_move_phase.argtypes = [C.POINTER(OrcState), C.c_uint64, _u32p, C.POINTER(C.c_int64)]
        L.orc_rebuild_occupancy.argtypes = [C.POINTER(OrcState)]
        L.orc_spawn_agents.restype = C.c_int
        L.orc_spawn_agents.argtypes = [C.c_int32, C.c_int32, _u8p, C.c_int64, C.c_uint64, _i32p, _i32p]
        L.orc_state_hash.restype = C.c_uint64
        L.orc_state_hash.argtypes = [C.POINTER(OrcState)]
        L.orc_trace.restype = C.c_int
        L.orc_trace.argtypes = [C.c_int32] * 6 + [_i32p, _i32p, C.c_int]
        L.orc_exp.restype = C.c_double
        L.orc_exp.argtypes = [C.c_double]
        _lib = L
    return _lib


def rng_u64(seed, agent, step, draw) -> int:
    return lib().orc_rng_u64(seed, agent, step, draw)


def unit_interval(x: int) -> float:
    return lib().orc_unit_interval(x)


def compute_blocksize(n: int, cores: int) -> int:
    return lib().orc_compute_blocksize(n, cores)


def static_field(cells: np.ndarray, boundary: int = 0) -> np.ndarray:
    h, w = cells.shape
    out = np.empty(h * w, np.float64)
    lib().orc_static_field(w, h, boundary, np.ascontiguousarray(cells, np.uint8).ravel(), out)
    return out.reshape(h, w)


def sample_index(weights, u: float) -> int:
    w = np.ascontiguousarray(weights, np.float64)
    return lib().orc_sample_index(w, len(w), u)


def movement_order(n: int, seed: int, step: int) -> np.ndarray:
    out = np.empty(max(n, 1), np.uint32)
    lib().orc_movement_order(n, seed, step, out)
    return out[:n]


def spawn_agents(cells: np.ndarray, n: int, seed: int):
    h, w = cells.shape
    x = np.empty(max(n, 1), np.int32)
    y = np.empty(max(n, 1), np.int32)
    rc = lib().orc_spawn_agents(w, h, np.ascontiguousarray(cells, np.uint8).ravel(), n, seed, x, y)
    if rc != 0:
        raise RuntimeError("spawn_agents: not enough free cells")
    return x[:n].copy(), y[:n].copy()


class State:
    """A SimState restated as numpy SoA arrays, stepped by the C oracle."""

    def __init__(self, cells, field, x, y, v_max, alive=None, boundary=0, step=0,
                 potential=0, drive_gradient=0.0):
        self.cells = np.ascontiguousarray(cells, np.uint8)
        self.h, self.w = self.cells.shape
        self.field = np.ascontiguousarray(field, np.float64).reshape(self.h, self.w)
        n = len(x)
        self.x = np.ascontiguousarray(x, np.int32).copy()
        self.y = np.ascontiguousarray(y, np.int32).copy()
        self.v_max = np.ascontiguousarray(np.broadcast_to(v_max, (n,)), np.int32).copy()
        self.alive = (np.ones(n, np.uint8) if alive is None
                      else np.ascontiguousarray(alive, np.uint8).copy())
        self.occ = np.full(self.h * self.w, -1, np.int32)
        self.dx = self.x.copy()
        self.dy = self.y.copy()
        self.s = OrcState()
        s = self.s
        s.width, s.height, s.boundary = self.w, self.h, boundary
        s.cells = self.cells.ctypes.data
        s.field = self.field.ctypes.data
        s.n = n
        s.x, s.y = self.x.ctypes.data, self.y.ctypes.data
        s.v_max, s.alive = self.v_max.ctypes.data, self.alive.ctypes.data
        s.occ = self.occ.ctypes.data
        s.desired_x, s.desired_y = self.dx.ctypes.data, self.dy.ctypes.data
        s.step = step
        s.potential = potential
        s.drive_gradient = drive_gradient
        lib().orc_rebuild_occupancy(C.byref(s))

    @property
    def n(self):
        return len(self.x)

    @property
    def step(self):
        return self.s.step

    @step.setter
    def step(self, v):
        self.s.step = v

    @property
    def alive_count(self):
        return self.s.alive_count

    def candidates(self, agent):
        cx = np.empty(128, np.int32)
        cy = np.empty(128, np.int32)
        n = lib().orc_enumerate_candidates(C.byref(self.s), agent, cx, cy)
        return list(zip(cx[:n].tolist(), cy[:n].tolist()))

    def weights(self, agent, k_s):
        w = np.empty(128, np.float64)
        cx = np.empty(128, np.int32)
        cy = np.empty(128, np.int32)
        n = lib().orc_choice_weights(C.byref(self.s), agent, k_s, w, cx, cy)
        return w[:n].copy(), cx[:n].copy(), cy[:n].copy()

    def plan(self, k_s, seed):
        lib().orc_plan_phase(C.byref(self.s), k_s, seed)

    def move(self, seed):
        ex = np.empty(self.n + 1, np.uint32)
        ne = C.c_int64(0)
        disp = lib().orc_move_phase(C.byref(self.s), seed, ex, C.byref(ne))
        return ex[: ne.value].copy(), disp

    def step_once(self, k_s, seed):
        self.plan(k_s, seed)
        ex, disp = self.move(seed)
        self.s.step += 1
        return ex, disp

    def hash(self):
        return lib().orc_state_hash(C.byref(self.s))


# ---------------------------------------------------------------- reference (oracle/_ref)

_ref = None


def have_reference() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not have_reference():
            raise RuntimeError("oracle/_ref/libfastped_ref.so not built (reference absent)")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_u64.restype = C.c_uint64
        L.ref_rng_u64.argtypes = [C.c_uint64] * 4
        L.ref_compute_blocksize.restype = C.c_int
        L.ref_compute_blocksize.argtypes = [C.c_int64, C.c_int]
        L.ref_sample_index.restype = C.c_size_t
        L.ref_sample_index.argtypes = [_f64p, C.c_size_t, C.c_double]
        L.ref_exp.restype = C.c_double
        L.ref_exp.argtypes = [C.c_double]
        L.ref_static_field.restype = C.c_int
        L.ref_static_field.argtypes = [C.c_int, C.c_int, C.c_int, _u8p, _f64p]
        L.ref_state_create.restype = C.c_void_p
        L.ref_state_create.argtypes = [C.c_int, C.c_int, C.c_double, C.c_int, _u8p, C.c_void_p,
                                       C.c_int, _i32p, _i32p, _i32p, _u8p, C.c_int64, C.c_int,
                                       C.c_double]
        L.ref_state_destroy.argtypes = [C.c_void_p]
        L.ref_set_step.argtypes = [C.c_void_p, C.c_int64]
        L.ref_get_step.restype = C.c_int64
        L.ref_get_step.argtypes = [C.c_void_p]
        L.ref_alive_count.restype = C.c_int64
        L.ref_alive_count.argtypes = [C.c_void_p]
        L.ref_state_hash.restype = C.c_uint64
        L.ref_state_hash.argtypes = [C.c_void_p]
        L.ref_get_agents.argtypes = [C.c_void_p, _i32p, _i32p, _u8p]
        L.ref_get_desired.argtypes = [C.c_void_p, _i32p, _i32p]
        L.ref_set_desired.argtypes = [C.c_void_p, _i32p, _i32p]
        L.ref_get_occupancy.argtypes = [C.c_void_p, _i32p]
        L.ref_plan_phase.restype = C.c_int
        L.ref_plan_phase.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_int]
        L.ref_move_phase.restype = C.c_int64
        L.ref_move_phase.argtypes = [C.c_void_p, C.c_uint64, _u32p, C.c_int64, C.POINTER(C.c_int64)]
        L.ref_run.restype = C.c_int
        L.ref_run.argtypes = [C.c_void_p, C.c_double, C.c_uint64, C.c_int, C.c_int] + \
            [C.POINTER(C.c_double)] * 3 + [C.POINTER(C.c_int64)] * 2
        L.ref_choice_weights.restype = C.c_int
        L.ref_choice_weights.argtypes = [C.c_void_p, C.c_uint32, C.c_double, _f64p, _i32p, _i32p, C.c_int]
        L.ref_choose_desired.restype = C.c_int
        L.ref_choose_desired.argtypes = [C.c_void_p, C.c_uint32, C.c_double, C.c_uint64,
                                         C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
        L.ref_spawn_agents.restype = C.c_int
        L.ref_spawn_agents.argtypes = [C.c_int, C.c_int, _u8p, C.c_int, C.c_int64, C.c_int,
                                       C.c_uint64, _i32p, _i32p]
        for name in ("ref_make_plaza", "ref_make_corridor"):
            fn = getattr(L, name)
            fn.restype = C.c_int
            fn.argtypes = [C.c_double, C.c_double if name.endswith("corridor") else C.c_int,
                           C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_void_p]
        L.ref_fundamental_diagram.restype = C.c_int
        L.ref_fundamental_diagram.argtypes = [C.c_int, C.c_int, C.c_double, _u8p, C.c_int, _f64p, C.c_int,
                                              C.c_uint64, C.c_int, C.c_int, C.c_double, _f64p, _f64p, _f64p]
        L.ref_capacity_from_table.restype = C.c_int
        L.ref_capacity_from_table.argtypes = [C.POINTER(C.c_int64), _f64p, C.c_int, C.c_double, C.c_int64,
                                              C.c_int64, C.POINTER(C.c_int64), _f64p]
        _ref = L
    return _ref


class RefState:
    """A reference SimState (make_state over the unmodified headers)."""

    def __init__(self, cells, field, x, y, v_max, alive=None, boundary=0, step=0,
                 potential=0, drive_gradient=0.0, cell_size=0.4):
        L = ref()
        cells = np.ascontiguousarray(cells, np.uint8)
        self.h, self.w = cells.shape
        n = len(x)
        self.n = n
        x = np.ascontiguousarray(x, np.int32)
        y = np.ascontiguousarray(y, np.int32)
        v = np.ascontiguousarray(np.broadcast_to(v_max, (n,)), np.int32)
        al = (np.ones(n, np.uint8) if alive is None else np.ascontiguousarray(alive, np.uint8))
        if n == 0:
            x = np.zeros(1, np.int32); y = np.zeros(1, np.int32)
            v = np.full(1, 4, np.int32); al = np.zeros(1, np.uint8)
        fptr = None
        if field is not None:
            self._field = np.ascontiguousarray(field, np.float64)
            fptr = self._field.ctypes.data
        self.p = L.ref_state_create(self.w, self.h, cell_size, boundary, cells.ravel(), fptr, n,
                                    x, y, v, al, step, potential, drive_gradient)
        if not self.p:
            raise ValueError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "p", None):
            ref().ref_state_destroy(self.p)
            self.p = None

    @property
    def step(self):
        return ref().ref_get_step(self.p)

    @step.setter
    def step(self, v):
        ref().ref_set_step(self.p, v)

    @property
    def alive_count(self):
        return ref().ref_alive_count(self.p)

    def agents(self):
        n = max(self.n, 1)
        x = np.empty(n, np.int32); y = np.empty(n, np.int32); a = np.empty(n, np.uint8)
        ref().ref_get_agents(self.p, x, y, a)
        return x[: self.n], y[: self.n], a[: self.n]

    def desired(self):
        n = max(self.n, 1)
        x = np.empty(n, np.int32); y = np.empty(n, np.int32)
        ref().ref_get_desired(self.p, x, y)
        return x[: self.n], y[: self.n]

    def set_desired(self, x, y):
        ref().ref_set_desired(self.p, np.ascontiguousarray(x, np.int32), np.ascontiguousarray(y, np.int32))

    def occupancy(self):
        o = np.empty(self.w * self.h, np.int32)
        ref().ref_get_occupancy(self.p, o)
        return o.reshape(self.h, self.w)

    def plan(self, k_s, seed, cores=1):
        if ref().ref_plan_phase(self.p, k_s, seed, cores) != 0:
            raise ValueError(ref().ref_last_error().decode())

    def move(self, seed):
        ex = np.empty(self.n + 1, np.uint32)
        ne = C.c_int64(0)
        disp = ref().ref_move_phase(self.p, seed, ex, self.n + 1, C.byref(ne))
        return ex[: ne.value].copy(), disp

    def step_once(self, k_s, seed, cores=1):
        self.plan(k_s, seed, cores)
        ex, disp = self.move(seed)
        self.step = self.step + 1
        return ex, disp

    def run(self, k_s, seed, steps, cores):
        w, p, m = C.c_double(), C.c_double(), C.c_double()
        e, d = C.c_int64(), C.c_int64()
        rc = ref().ref_run(self.p, k_s, seed, steps, cores, C.byref(w), C.byref(p), C.byref(m),
                           C.byref(e), C.byref(d))
        if rc != 0:
            raise ValueError(ref().ref_last_error().decode())
        return dict(wall_time_s=w.value, plan_time_s=p.value, move_time_s=m.value,
                    exited=e.value, displacement_cells=d.value)

    def weights(self, agent, k_s):
        w = np.empty(128, np.float64); cx = np.empty(128, np.int32); cy = np.empty(128, np.int32)
        n = ref().ref_choice_weights(self.p, agent, k_s, w, cx, cy, 128)
        return w[:n].copy(), cx[:n].copy(), cy[:n].copy()

    def hash(self):
        return ref().ref_state_hash(self.p)


def ref_fundamental_diagram(cells, cell_size, v_max, densities, seed, warmup=100, measure=296,
                            drive_gradient=8.0):
    """The reference's fundamental_diagram (bench.hpp:244-305) on a periodic-x corridor:
    (density, mean_speed, flow) arrays."""
    cells = np.ascontiguousarray(cells, np.uint8)
    h, w = cells.shape
    d = np.ascontiguousarray(densities, np.float64)
    out = [np.empty(len(d), np.float64) for _ in range(3)]
    if ref().ref_fundamental_diagram(w, h, cell_size, cells.ravel(), v_max, d, len(d), seed, warmup, measure,
                                     drive_gradient, *out) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_capacity_from_table(ns, ts, budget, start_n=1000, max_n=(2 ** 63 - 1) // 2):
    """The reference's realtime_capacity (bench.hpp:162-208) over a (n -> wall time) table:
    dict of its CapacityResult fields plus the number of probes it made."""
    ns = np.ascontiguousarray(ns, np.int64)
    ts = np.ascontiguousarray(ts, np.float64)
    o6 = np.zeros(6, np.int64)
    o3 = np.zeros(3, np.float64)
    if ref().ref_capacity_from_table(ns.ctypes.data_as(C.POINTER(C.c_int64)), ts, len(ns), budget, start_n, max_n,
                                     o6.ctypes.data_as(C.POINTER(C.c_int64)), o3) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return dict(capacity=int(o6[0]), n_low=int(o6[1]), n_high=int(o6[2]), below_start=bool(o6[3]),
                capped=bool(o6[4]), probes=int(o6[5]), t_low_s=float(o3[0]), t_high_s=float(o3[1]),
                budget_s=float(o3[2]))


def ref_static_field(cells, boundary=0):
    cells = np.ascontiguousarray(cells, np.uint8)
    h, w = cells.shape
    out = np.empty(h * w, np.float64)
    if ref().ref_static_field(w, h, boundary, cells.ravel(), out) != 0:
        raise ValueError(ref().ref_last_error().decode())
    return out.reshape(h, w)


def physical_core_count() -> int:
    """Unique (physical id, core id) pairs, as tests/acceptance.cpp:25-44 counts them."""
    seen = set()
    phys = -1
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if ":" not in line:
                    continue
                key, _, val = line.partition(":")
                key = key.strip()
                if key == "physical id":
                    phys = int(val)
                elif key == "core id":
                    seen.add((phys, int(val)))
    except OSError:
        pass
    return len(seen) if seen else (os.cpu_count() or 1)
