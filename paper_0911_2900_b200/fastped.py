"""Python mirror of the reference's `namespace fastped` API over the CUDA C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/fastped/*.hpp
(cited per function).  Geometry and rosters are numpy arrays; every compute call goes through
paper_0911_2900_b200/libfastped_b200.so (include/fastped_b200.h).  There is no CPU fallback:
on a box without a usable GPU the compute calls raise ``DeviceError``.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libfastped_b200.so")
# experiments only: another build of the library (tools/build_variant.py); never set in product runs
_LIB_OVERRIDE = os.environ.get("FASTPED_B200_LIB")

FREE, WALL, EXIT = 0, 1, 2                      # CellKind, world.hpp:18
CLOSED, PERIODIC_X = 0, 1                       # Boundary, world.hpp:19
EXIT_DISTANCE, DRIVE_X = 0, 1                   # Potential, state.hpp:17
K_MIN_VMAX, K_MAX_VMAX = 1, 5                   # agents.hpp:9-10
K_DEFAULT_DRIVE_GRADIENT = 8.0                  # bench.hpp:238

FP_OK, FP_EINVAL, FP_ERUNTIME, FP_ECUDA, FP_ENCCL = 0, 1, 2, 3, 4


class DeviceError(RuntimeError):
    """CUDA unavailable or failed (FP_ECUDA).  Never silently replaced by a CPU path."""


class _Grid(C.Structure):
    _fields_ = [("width", C.c_int32), ("height", C.c_int32), ("cell_size", C.c_double),
                ("boundary", C.c_int32)]


class _StepStats(C.Structure):
    _fields_ = [("alive", C.c_int64), ("exited", C.c_int64), ("displacement_cells", C.c_int64)]


class _RunStats(C.Structure):
    _fields_ = [("wall_time_s", C.c_double), ("plan_time_s", C.c_double), ("move_time_s", C.c_double),
                ("steps", C.c_int64), ("exited", C.c_int64), ("displacement_cells", C.c_int64),
                ("alive", C.c_int64), ("agent_updates", C.c_int64)]


class _Counters(C.Structure):
    _fields_ = [("kernel_launches", C.c_int64), ("motion_rounds", C.c_int64),
                ("plan_fallbacks", C.c_int64), ("planned_agents", C.c_int64),
                ("motion_seed_ns", C.c_int64), ("motion_grid_ns", C.c_int64),
                ("motion_tail_ns", C.c_int64), ("motion_grid_rounds", C.c_int64),
                ("motion_mark_ns", C.c_int64), ("motion_contended", C.c_int64),
                ("motion_prep_ns", C.c_int64)]


_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")

# name -> (restype, argtypes); the complete export list of include/fastped_b200.h
SIGNATURES = {
    "fp_version": (C.c_char_p, []),
    "fp_last_error": (C.c_char_p, [C.c_void_p]),
    "fp_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "fp_compute_blocksize": (C.c_int, [C.c_int64, C.c_int, C.POINTER(C.c_int32)]),
    "fp_create": (C.c_int, [C.POINTER(_Grid), _u8p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "fp_destroy": (None, [C.c_void_p]),
    "fp_static_field": (C.c_int, [C.POINTER(_Grid), _u8p, C.c_int, _f64p]),
    "fp_get_field": (C.c_int, [C.c_void_p, _f64p]),
    "fp_set_agents": (C.c_int, [C.c_void_p, C.c_uint32, _i32p, _i32p, _i32p, C.c_void_p, C.c_int64]),
    "fp_update_agents": (C.c_int, [C.c_void_p, _i32p, _i32p, C.c_void_p]),
    "fp_set_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "fp_get_step": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "fp_get_alive_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "fp_get_last_dx": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "fp_get_run_dx": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "fp_set_potential": (C.c_int, [C.c_void_p, C.c_int, C.c_double]),
    "fp_set_desired": (C.c_int, [C.c_void_p, _i32p, _i32p]),
    "fp_plan": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64]),
    "fp_move": (C.c_int, [C.c_void_p, C.c_uint64, C.POINTER(_StepStats)]),
    "fp_step": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.POINTER(_StepStats)]),
    "fp_run": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_int32, C.POINTER(_RunStats)]),
    "fp_get_agents": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "fp_get_desired": (C.c_int, [C.c_void_p, _i32p, _i32p]),
    "fp_get_occupancy": (C.c_int, [C.c_void_p, _i32p]),
    "fp_get_exited": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.POINTER(C.c_uint32)]),
    "fp_get_order": (C.c_int, [C.c_void_p, _u32p, C.c_uint32, C.POINTER(C.c_uint32)]),
    "fp_state_hash": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "fp_hash_roster": (C.c_int, [C.c_int64, C.c_int64, C.c_uint32, _i32p, _i32p, _u8p, C.POINTER(C.c_uint64)]),
    "fp_get_choice": (C.c_int, [C.c_void_p, C.c_uint32, C.c_double, _i32p, _i32p, _f64p, _f32p,
                                C.c_uint32, C.POINTER(C.c_uint32)]),
    "fp_choose_desired": (C.c_int, [C.c_void_p, C.c_uint32, C.c_int32, C.c_int32, C.c_int32, C.c_int64, C.c_double,
                                    C.c_uint64, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fp_enumerate_candidates": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, _i32p, _i32p, C.c_uint32,
                                          C.POINTER(C.c_uint32)]),
    "fp_movement_order": (C.c_int, [C.c_int64, C.c_uint64, C.c_int64, C.c_int, _u32p]),
    "fp_spawn_agents": (C.c_int, [C.c_int32, C.c_int32, _u8p, C.c_int64, C.c_uint64, _i32p, _i32p]),
    "fp_get_counters": (C.c_int, [C.c_void_p, C.POINTER(_Counters)]),
    "fp_time_plan_kernel": (C.c_int, [C.c_void_p, C.c_double, C.c_uint64, C.c_int32, C.POINTER(C.c_double)]),
    # multi-GPU x strips (strip.cu)
    "fp_strip_bounds": (C.c_int, [C.c_int32, C.c_int, C.c_int, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "fp_strip_config": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int32, C.c_int32, C.c_uint32, C.c_uint32]),
    "fp_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "fp_strip_set_nccl": (C.c_int, [C.c_void_p, C.c_void_p]),
    "fp_strip_set_exchange": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fp_strips_step": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.POINTER(_StepStats)]),
    "fp_strips_run": (C.c_int, [C.c_void_p, C.c_int, C.c_double, C.c_uint64, C.c_int32, C.POINTER(_RunStats)]),
    "fp_strip_get_owned": (C.c_int, [C.c_void_p, _u8p]),
}

_lib = None


def library():
    """Loads the in-tree CUDA library (building it first if it is missing or stale)."""
    global _lib
    if _lib is None:
        if _LIB_OVERRIDE:
            L = C.CDLL(_LIB_OVERRIDE)
        else:
            from . import build as _build
            _build.build()
            L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(rc: int, ctx=None):
    if rc == FP_OK:
        return
    msg = (library().fp_last_error(ctx) or b"").decode()
    if rc == FP_EINVAL:
        raise ValueError(msg)
    if rc == FP_ERUNTIME:
        raise RuntimeError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------------------------- geometry
@dataclass
class Grid:
    """Immutable scenario geometry (world.hpp:35-121); cells is an HxW uint8 CellKind array."""
    cells: np.ndarray
    cell_size: float = 0.4
    boundary: int = CLOSED

    def __post_init__(self):
        self.cells = np.ascontiguousarray(self.cells, np.uint8)
        if self.cells.ndim != 2 or self.cells.size == 0:
            raise ValueError("Grid: width and height must be >= 1")
        if not self.cell_size > 0.0:
            raise ValueError("Grid: cell_size must be > 0")
        c = self.cells
        if self.boundary == CLOSED:
            border = np.concatenate([c[0], c[-1], c[:, 0], c[:, -1]])
            if (border == FREE).any():
                raise ValueError("Grid: closed boundary requires every border cell to be Wall or Exit")
        elif (c[0] != WALL).any() or (c[-1] != WALL).any():
            raise ValueError("Grid: periodic-x boundary requires solid top and bottom rows")

    @property
    def width(self) -> int:
        return self.cells.shape[1]

    @property
    def height(self) -> int:
        return self.cells.shape[0]

    def free_cell_count(self) -> int:
        return int((self.cells == FREE).sum())

    def exit_cell_count(self) -> int:
        return int((self.cells == EXIT).sum())

    def desc(self) -> _Grid:
        return _Grid(self.width, self.height, self.cell_size, self.boundary)


def from_rows(rows: Sequence[str], boundary: int = CLOSED, cell_size: float = 0.4) -> Grid:
    """The tests' from_rows helper (tests/test_planning.cpp:15-24): '#' Wall, 'E' Exit, else Free."""
    table = {"#": WALL, "E": EXIT}
    cells = np.array([[table.get(ch, FREE) for ch in r] for r in rows], np.uint8)
    return Grid(cells, cell_size, boundary)


def make_plaza(side_m: float, exits: int, cell_size: float = 0.4, width: Optional[int] = None,
               height: Optional[int] = None) -> Grid:
    """make_plaza (scenario_io.hpp:74-105); width/height generalise it to W != H (config 4)."""
    n = int(round(side_m / cell_size))
    w = width if width is not None else n
    h = height if height is not None else n
    if w < 3 or h < 3:
        raise ValueError("make_plaza: side must be at least 3 cells, got %d" % min(w, h))
    if exits < 0:
        raise ValueError("make_plaza: exits must be >= 0")
    cells = np.zeros((h, w), np.uint8)
    cells[0, :] = WALL
    cells[-1, :] = WALL
    cells[:, 0] = WALL
    cells[:, -1] = WALL
    ring = ([(x, 0) for x in range(1, w - 1)] + [(w - 1, y) for y in range(1, h - 1)] +
            [(x, h - 1) for x in range(w - 2, 0, -1)] + [(0, y) for y in range(h - 2, 0, -1)])
    if exits > len(ring):
        raise ValueError("make_plaza: more exits than non-corner border cells")
    for k in range(exits):
        x, y = ring[(2 * k + 1) * len(ring) // (2 * exits)]
        cells[y, x] = EXIT
    return Grid(cells, cell_size, CLOSED)


def make_corridor(length_m: float, width_m: float, cell_size: float = 0.4) -> Grid:
    """make_corridor (scenario_io.hpp:109-121): periodic-x, solid top/bottom rows, no exits."""
    w = int(round(length_m / cell_size))
    h = int(round(width_m / cell_size))
    if w < 3 or h < 3:
        raise ValueError("make_corridor: corridor must be at least 3x3 cells, got %dx%d" % (w, h))
    cells = np.zeros((h, w), np.uint8)
    cells[0, :] = WALL
    cells[-1, :] = WALL
    return Grid(cells, cell_size, PERIODIC_X)


def compute_static_field(grid: Grid, device: int = 0) -> np.ndarray:
    """compute_static_field (world.hpp:220-266) on the device; bit-identical fp64 field."""
    out = np.empty(grid.height * grid.width, np.float64)
    g = grid.desc()
    _check(library().fp_static_field(C.byref(g), grid.cells.ravel(), device, out))
    return out.reshape(grid.height, grid.width)


@dataclass
class Scenario:
    """Named geometry plus its exit-distance field (scenario_io.hpp:21-25)."""
    name: str
    grid: Grid
    field: np.ndarray


def make_scenario(name: str, grid: Grid, device: int = 0) -> Scenario:
    return Scenario(name, grid, compute_static_field(grid, device))


@dataclass
class Roster:
    """A roster of agents in SoA form (agents.hpp:13-18): ids are the indices."""
    x: np.ndarray
    y: np.ndarray
    v_max: np.ndarray
    alive: np.ndarray

    def __len__(self):
        return len(self.x)


def roster(positions: Sequence, v_max=4) -> Roster:
    p = np.asarray(list(positions), np.int32).reshape(-1, 2)
    n = len(p)
    return Roster(p[:, 0].copy(), p[:, 1].copy(), np.broadcast_to(np.asarray(v_max, np.int32), (n,)).copy(),
                  np.ones(n, np.uint8))


def spawn_agents(grid: Grid, n: int, v_max: int, seed: int) -> Roster:
    """spawn_agents (scenario_io.hpp:47-69)."""
    if n < 0:
        raise ValueError("spawn_agents: agent count must be >= 0")
    if not K_MIN_VMAX <= v_max <= K_MAX_VMAX:
        raise ValueError("spawn_agents: v_max must be in [1,5]")
    x = np.empty(max(n, 1), np.int32)
    y = np.empty(max(n, 1), np.int32)
    _check(library().fp_spawn_agents(grid.width, grid.height, grid.cells.ravel(), n, seed, x, y))
    return Roster(x[:n].copy(), y[:n].copy(), np.full(n, v_max, np.int32), np.ones(n, np.uint8))


# ---------------------------------------------------------------------------------- params
@dataclass
class SimParams:
    """agents.hpp:22-45."""
    k_s: float = 1.2
    k_other: float = 0.0
    v_max: int = 4
    seed: int = 1
    steps: int = 396
    dt: float = 1.0

    def validate(self):
        if self.k_other != 0.0:
            raise ValueError("SimParams: k_other must be 0")
        if not K_MIN_VMAX <= self.v_max <= K_MAX_VMAX:
            raise ValueError("SimParams: v_max must be in [1,5]")
        if self.steps < 1:
            raise ValueError("SimParams: steps must be >= 1")
        if not self.dt > 0.0:
            raise ValueError("SimParams: dt must be > 0")


@dataclass
class ScheduleParams:
    """engine.hpp:21-23.  `cores` is kept for API compatibility (it never changes results)."""
    cores: int = 1


def compute_blocksize(number_of_agents: int, cores: int) -> int:
    """engine.hpp:27-33."""
    out = C.c_int32()
    _check(library().fp_compute_blocksize(number_of_agents, cores, C.byref(out)))
    return out.value


@dataclass
class MoveOutcome:
    exited: List[int]
    displacement_cells: int


@dataclass
class StepStats:
    alive: int
    exited: int
    displacement_cells: int


@dataclass
class RunStats:
    wall_time_s: float
    plan_time_s: float
    move_time_s: float
    steps: int
    exited: int
    displacement_cells: int
    alive: int
    agent_updates: int


# ---------------------------------------------------------------------------------- state
class SimState:
    """Device-resident SimState (state.hpp:22-36): grid, field, roster, occupancy, step."""

    def __init__(self, grid: Grid, field: Optional[np.ndarray], rost: Roster, device: int = 0,
                 step: int = 0):
        L = library()
        self.grid = grid
        self.n = len(rost)
        self._ctx = C.c_void_p()
        g = grid.desc()
        fptr = None
        if field is not None:
            self._field = np.ascontiguousarray(field, np.float64)
            if self._field.size != grid.width * grid.height:
                raise ValueError("make_state: field dimensions do not match grid")
            fptr = self._field.ctypes.data
        _check(L.fp_create(C.byref(g), grid.cells.ravel(), fptr, device, C.byref(self._ctx)))
        x = np.ascontiguousarray(rost.x, np.int32)
        y = np.ascontiguousarray(rost.y, np.int32)
        v = np.ascontiguousarray(rost.v_max, np.int32)
        a = np.ascontiguousarray(rost.alive, np.uint8)
        if self.n == 0:
            x = y = v = np.zeros(1, np.int32)
        _check(L.fp_set_agents(self._ctx, self.n, x, y, v, a.ctypes.data if self.n else None, step),
               self._ctx)
        self.potential = EXIT_DISTANCE
        self.drive_gradient = 0.0

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            library().fp_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- potential
    def set_potential(self, kind: int, drive_gradient: float = 0.0):
        self.potential = kind
        self.drive_gradient = drive_gradient
        _check(library().fp_set_potential(self._ctx, kind, drive_gradient), self._ctx)

    # -- step counter
    @property
    def step(self) -> int:
        v = C.c_int64()
        _check(library().fp_get_step(self._ctx, C.byref(v)), self._ctx)
        return v.value

    @step.setter
    def step(self, s: int):
        _check(library().fp_set_step(self._ctx, s), self._ctx)

    @property
    def alive(self) -> int:
        v = C.c_int64()
        _check(library().fp_get_alive_count(self._ctx, C.byref(v)), self._ctx)
        return v.value

    @property
    def last_dx(self) -> int:
        """Sum of segment_dx(x before, x after) over all agents in the last move phase."""
        v = C.c_int64()
        _check(library().fp_get_last_dx(self._ctx, C.byref(v)), self._ctx)
        return v.value

    @property
    def run_dx(self) -> int:
        """Sum of segment_dx over every step of the last run()."""
        v = C.c_int64()
        _check(library().fp_get_run_dx(self._ctx, C.byref(v)), self._ctx)
        return v.value

    # -- dumps
    def agents(self, out=None):
        """(x, y, alive) of every agent; `out` = three caller-owned (e.g. pinned) arrays to fill."""
        if out is None:
            n = max(self.n, 1)
            x = np.empty(n, np.int32)
            y = np.empty(n, np.int32)
            a = np.empty(n, np.uint8)
        else:
            x, y, a = out
            if not (x.dtype == np.int32 and y.dtype == np.int32 and a.dtype == np.uint8 and len(x) >= self.n
                    and len(y) >= self.n and len(a) >= self.n and x.flags.c_contiguous and y.flags.c_contiguous
                    and a.flags.c_contiguous):
                raise ValueError("agents(out=...): need contiguous int32, int32, uint8 arrays of n elements")
        _check(library().fp_get_agents(self._ctx, x.ctypes.data, y.ctypes.data, a.ctypes.data), self._ctx)
        return x[: self.n], y[: self.n], a[: self.n]

    def set_agents(self, x, y, alive):
        _check(library().fp_update_agents(self._ctx, np.ascontiguousarray(x, np.int32),
                                          np.ascontiguousarray(y, np.int32),
                                          np.ascontiguousarray(alive, np.uint8).ctypes.data), self._ctx)

    def desired(self):
        n = max(self.n, 1)
        x = np.empty(n, np.int32)
        y = np.empty(n, np.int32)
        _check(library().fp_get_desired(self._ctx, x, y), self._ctx)
        return x[: self.n], y[: self.n]

    def set_desired(self, x, y):
        _check(library().fp_set_desired(self._ctx, np.ascontiguousarray(x, np.int32),
                                        np.ascontiguousarray(y, np.int32)), self._ctx)

    def occupancy(self) -> np.ndarray:
        o = np.empty(self.grid.width * self.grid.height, np.int32)
        _check(library().fp_get_occupancy(self._ctx, o), self._ctx)
        return o.reshape(self.grid.height, self.grid.width)

    def field(self) -> np.ndarray:
        o = np.empty(self.grid.width * self.grid.height, np.float64)
        _check(library().fp_get_field(self._ctx, o), self._ctx)
        return o.reshape(self.grid.height, self.grid.width)

    def last_order(self) -> np.ndarray:
        n = C.c_uint32()
        buf = np.empty(max(self.n, 1), np.uint32)
        _check(library().fp_get_order(self._ctx, buf, len(buf), C.byref(n)), self._ctx)
        return buf[: n.value].copy()

    def choice(self, agent: int, k_s: float):
        """Candidates, exact weights and production choice probabilities of one agent."""
        cx = np.empty(128, np.int32)
        cy = np.empty(128, np.int32)
        w = np.empty(128, np.float64)
        p = np.empty(128, np.float32)
        n = C.c_uint32()
        _check(library().fp_get_choice(self._ctx, agent, k_s, cx, cy, w, p, 128, C.byref(n)), self._ctx)
        k = n.value
        return cx[:k].copy(), cy[:k].copy(), w[:k].copy(), p[:k].copy()

    def time_plan_kernel(self, k_s: float, seed: int, iters: int = 10) -> float:
        """Average plan-kernel launch duration in ms (CUDA events), for the roofline."""
        ms = C.c_double()
        _check(library().fp_time_plan_kernel(self._ctx, k_s, seed, iters, C.byref(ms)), self._ctx)
        return ms.value

    def counters(self) -> dict:
        c = _Counters()
        _check(library().fp_get_counters(self._ctx, C.byref(c)), self._ctx)
        return {k: getattr(c, k) for k, _ in _Counters._fields_}


def make_state(scenario_or_grid, rost: Roster, field: Optional[np.ndarray] = None, device: int = 0) -> SimState:
    """make_state (state.hpp:38-76 / scenario_io.hpp:41-43)."""
    if isinstance(scenario_or_grid, Scenario):
        return SimState(scenario_or_grid.grid, scenario_or_grid.field, rost, device)
    return SimState(scenario_or_grid, field, rost, device)


def plan_phase(st: SimState, params: SimParams, sched: ScheduleParams = ScheduleParams()):
    """plan_phase (engine.hpp:71-84)."""
    if sched.cores < 1:
        raise ValueError("plan_phase: cores must be >= 1")
    _check(library().fp_plan(st._ctx, params.k_s, params.seed), st._ctx)


def move_phase(st: SimState, params: SimParams) -> MoveOutcome:
    """move_phase (engine.hpp:95-135)."""
    s = _StepStats()
    _check(library().fp_move(st._ctx, params.seed, C.byref(s)), st._ctx)
    n = C.c_uint32()
    buf = np.empty(max(s.exited, 1), np.uint32)
    _check(library().fp_get_exited(st._ctx, buf, len(buf), C.byref(n)), st._ctx)
    return MoveOutcome(buf[: n.value].tolist(), s.displacement_cells)


def step(st: SimState, params: SimParams, sched: ScheduleParams = ScheduleParams()) -> StepStats:
    """step (engine.hpp:143-148)."""
    if sched.cores < 1:
        raise ValueError("plan_phase: cores must be >= 1")
    s = _StepStats()
    _check(library().fp_step(st._ctx, params.k_s, params.seed, C.byref(s)), st._ctx)
    return StepStats(s.alive, s.exited, s.displacement_cells)


def run(st: SimState, params: SimParams, sched: ScheduleParams = ScheduleParams()) -> RunStats:
    """run (engine.hpp:161-183): device loop, CUDA-event timed."""
    params.validate()
    if sched.cores < 1:
        raise ValueError("run: cores must be >= 1")
    r = _RunStats()
    _check(library().fp_run(st._ctx, params.k_s, params.seed, params.steps, C.byref(r)), st._ctx)
    return RunStats(r.wall_time_s, r.plan_time_s, r.move_time_s, r.steps, r.exited,
                    r.displacement_cells, r.alive, r.agent_updates)


def state_hash(st: SimState) -> int:
    """state_hash (state.hpp:80-95)."""
    h = C.c_uint64()
    _check(library().fp_state_hash(st._ctx, C.byref(h)), st._ctx)
    return h.value


def movement_order(n: int, seed: int, step_index: int, device: int = 0) -> np.ndarray:
    """The device Fisher-Yates permutation of positions 0..n-1 (engine.hpp:99-111)."""
    out = np.empty(max(n, 1), np.uint32)
    _check(library().fp_movement_order(n, seed, step_index, device, out))
    return out[:n].copy()


def cuda_available() -> bool:
    try:
        import torch  # noqa: F401  (plumbing only: device query)
        return bool(torch.cuda.is_available())
    except Exception:
        return False


# ---------------------------------------------------------------------------------- x strips
# One simulation decomposed over N x-strips (strip.cu): rank r owns
# the agents standing in columns strip_bounds(W, r, N); the step equals the 1-GPU step bit for
# bit.  StripSet drives all ranks from this process (device-to-device exchange: virtual strips
# on one GPU, or one context per GPU); StripRank is one rank of a multi-process job whose
# exchange is NCCL (one process per GPU) or a host allgather callback (e.g. torch gloo).

def strip_bounds(width: int, rank: int, nranks: int):
    lo, hi = C.c_int32(), C.c_int32()
    _check(library().fp_strip_bounds(width, rank, nranks, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


class StripRank(SimState):
    """One strip rank: the global grid, field and roster, plus its strip.  `exchange` is
    "nccl" (nccl_id: 128 bytes from nccl_unique_id(), shared by the ranks) or a Python callable
    allgather(send: bytes-like memoryview, recv: memoryview of N * len(send)) for the host
    transport."""

    def __init__(self, grid: Grid, field, rost: Roster, rank: int, nranks: int, device: int = 0,
                 exchange=None, nccl_id: Optional[bytes] = None, cap_deferred: int = 0, cap_exits: int = 0,
                 x_bounds=None):
        super().__init__(grid, field, rost, device)
        self.rank, self.nranks = rank, nranks
        lo, hi = x_bounds if x_bounds is not None else strip_bounds(grid.width, rank, nranks)
        self.x_lo, self.x_hi = lo, hi
        L = library()
        _check(L.fp_strip_config(self._ctx, rank, nranks, lo, hi, cap_deferred, cap_exits), self._ctx)
        self._cb = None
        if nccl_id is not None:
            buf = C.create_string_buffer(bytes(nccl_id), 128)
            _check(L.fp_strip_set_nccl(self._ctx, buf), self._ctx)
        elif exchange is not None:
            AG = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p)

            def _cb(user, send, nbytes, recv):
                try:
                    exchange(memoryview((C.c_char * nbytes).from_address(send)).cast("B"),
                             memoryview((C.c_char * (nbytes * nranks)).from_address(recv)).cast("B"))
                    return 0
                except Exception:  # noqa: BLE001 -- reported through the status code
                    import traceback
                    traceback.print_exc()
                    return 1

            self._cb = AG(_cb)
            _check(L.fp_strip_set_exchange(self._ctx, C.cast(self._cb, C.c_void_p), None), self._ctx)

    def owned(self) -> np.ndarray:
        o = np.empty(max(self.n, 1), np.uint8)
        _check(library().fp_strip_get_owned(self._ctx, o), self._ctx)
        return o[: self.n]


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(library().fp_nccl_unique_id(buf))
    return buf.raw


def merge_strip_agents(parts):
    """(x, y, alive) of the whole roster from every rank's (x, y, alive, owned): each agent from
    the rank that owns it (alive or exited there); agents no rank owns (exited in a resolved
    walk, or dead from the start) hold identical positions on every rank."""
    x, y, a, _ = (np.array(v) for v in parts[0])
    for px, py, pa, po in parts:
        sel = po.astype(bool)
        x[sel], y[sel], a[sel] = px[sel], py[sel], pa[sel]
    return x, y, a


def hash_roster(step: int, alive_count: int, x, y, a) -> int:
    """state_hash (state.hpp:80-95) of a roster given as host arrays."""
    h = C.c_uint64()
    n = len(x)
    x = np.ascontiguousarray(x, np.int32) if n else np.zeros(1, np.int32)
    y = np.ascontiguousarray(y, np.int32) if n else np.zeros(1, np.int32)
    a = np.ascontiguousarray(a, np.uint8) if n else np.zeros(1, np.uint8)
    _check(library().fp_hash_roster(step, alive_count, n, x, y, a, C.byref(h)))
    return h.value


class StripSet:
    """All N strip ranks of one simulation in this process (fp_strips_step / fp_strips_run).
    devices: one CUDA ordinal per rank (default: all on device 0 -- virtual strips)."""

    def __init__(self, grid: Grid, field, rost: Roster, nranks: int, devices=None, cap_deferred: int = 0,
                 cap_exits: int = 0, x_bounds=None):
        devices = devices or [0] * nranks
        self.grid, self.n, self.nranks = grid, len(rost), nranks
        self.ranks = []
        for r in range(nranks):
            st = SimState(grid, field, rost, devices[r])
            lo, hi = x_bounds[r] if x_bounds is not None else strip_bounds(grid.width, r, nranks)
            _check(library().fp_strip_config(st._ctx, r, nranks, lo, hi, cap_deferred, cap_exits), st._ctx)
            self.ranks.append(st)
        self._arr = (C.c_void_p * nranks)(*[st._ctx.value for st in self.ranks])

    def set_potential(self, kind: int, drive_gradient: float = 0.0):
        for st in self.ranks:
            st.set_potential(kind, drive_gradient)

    def step(self, params: SimParams) -> StepStats:
        s = _StepStats()
        _check(library().fp_strips_step(self._arr, self.nranks, params.k_s, params.seed, C.byref(s)),
               self.ranks[0]._ctx)
        return StepStats(s.alive, s.exited, s.displacement_cells)

    def run(self, params: SimParams) -> RunStats:
        params.validate()
        r = _RunStats()
        _check(library().fp_strips_run(self._arr, self.nranks, params.k_s, params.seed, params.steps, C.byref(r)),
               self.ranks[0]._ctx)
        return RunStats(r.wall_time_s, r.plan_time_s, r.move_time_s, r.steps, r.exited,
                        r.displacement_cells, r.alive, r.agent_updates)

    def exited(self):
        n = C.c_uint32()
        buf = np.empty(max(self.n, 1), np.uint32)
        _check(library().fp_get_exited(self.ranks[0]._ctx, buf, len(buf), C.byref(n)), self.ranks[0]._ctx)
        return buf[: n.value].tolist()

    def agents(self):
        parts = []
        for st in self.ranks:
            x, y, a = st.agents()
            o = np.empty(max(self.n, 1), np.uint8)
            _check(library().fp_strip_get_owned(st._ctx, o), st._ctx)
            parts.append((x.copy(), y.copy(), a.copy(), o[: self.n]))
        return merge_strip_agents(parts)

    @property
    def step_index(self) -> int:
        return self.ranks[0].step

    @property
    def alive(self) -> int:
        return self.ranks[0].alive

    def state_hash(self) -> int:
        x, y, a = self.agents()
        return hash_roster(self.step_index, self.alive, x, y, a)

    def close(self):
        for st in self.ranks:
            st.close()
