"""Measurement harness on the device engine.

Restates the reference's harness (fastped/bench.hpp, fastped/scenario_io.hpp) over this
package's engine: the (cores, agents, v_max) sweep and its speed factors, the real-time capacity
search, the fundamental-diagram measurement on a periodic corridor with the Weidmann comparison,
and the reference's CSV schemas byte for byte.  Every simulation runs on the GPU through the
C ABI; the fundamental diagram's per-step x displacement is reduced on the device during the
walks (`SimState.last_dx`) instead of diffing downloaded positions.  `cores` is kept wherever
the reference has it (validated, recorded) -- it never changes device results, as it never
changes the reference's.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Sequence, Tuple

from . import fastped as fp

K_DEFAULT_DRIVE_GRADIENT = fp.K_DEFAULT_DRIVE_GRADIENT  # bench.hpp:238

# Kladek-form reference curve, Weidmann parameters (bench.hpp:323-326)
WEIDMANN_FREE_SPEED = 1.34  # m/s
WEIDMANN_GAMMA = 1.913  # m^-2
WEIDMANN_MAX_DENSITY = 5.4  # m^-2

RUN_CSV_HEADER = "scenario,agents_initial,v_max,cores,steps,wall_time_s,plan_time_s,move_time_s,seed"
SPEEDUP_CSV_HEADER = "scenario,agents_initial,v_max,cores,wall_time_s,factor"
FD_CSV_HEADER = "density,mean_speed,flow"


# ---------------------------------------------------------------------------------- records / CSV
@dataclass
class RunRecord:
    """One benchmark measurement row (scenario_io.hpp:123-133)."""
    scenario: str
    agents_initial: int = 0
    v_max: int = 0
    cores: int = 0
    steps: int = 0
    wall_time_s: float = 0.0
    plan_time_s: float = 0.0
    move_time_s: float = 0.0
    seed: int = 0


def _fixed6(v: float) -> str:
    return "%.6f" % v  # detail::append_fixed6 (scenario_io.hpp:141-145)


def _check_csv_text(name: str):
    """detail::check_csv_text (scenario_io.hpp:147-151)."""
    if "," in name or "\n" in name:
        raise ValueError("csv: scenario name must not contain ',' or newline: " + name)


def runs_to_csv(records: Sequence[RunRecord]) -> str:
    """to_csv(vector<RunRecord>) (scenario_io.hpp:157-177): pinned header, 6 fractional digits
    on times, '\\n' endings, exactly one trailing '\\n'."""
    out = [RUN_CSV_HEADER]
    for r in records:
        _check_csv_text(r.scenario)
        out.append("%s,%d,%d,%d,%d,%s,%s,%s,%d" % (r.scenario, r.agents_initial, r.v_max, r.cores, r.steps,
                                                   _fixed6(r.wall_time_s), _fixed6(r.plan_time_s),
                                                   _fixed6(r.move_time_s), r.seed))
    return "\n".join(out) + "\n"


def parse_run_csv(text: str) -> List[RunRecord]:
    """parse_run_csv (scenario_io.hpp:219-243)."""
    lines = text.split("\n")
    if not lines or lines[0] != RUN_CSV_HEADER:
        raise RuntimeError("csv: missing or unexpected header")
    records = []
    for i, line in enumerate(lines[1:], start=1):
        if not line:
            continue  # trailing newline
        f = line.split(",")
        if len(f) != 9:
            raise RuntimeError("csv row %d: expected 9 fields, got %d" % (i + 1, len(f)))
        try:
            records.append(RunRecord(f[0], int(f[1]), int(f[2]), int(f[3]), int(f[4]), float(f[5]), float(f[6]),
                                     float(f[7]), int(f[8])))
        except ValueError:
            raise RuntimeError("csv row %d: malformed number" % (i + 1)) from None
    return records


# ---------------------------------------------------------------------------------- sweep
@dataclass
class SweepSpec:
    """bench.hpp:25-46."""
    cores_list: List[int] = field(default_factory=list)
    agents_list: List[int] = field(default_factory=list)
    vmax_list: List[int] = field(default_factory=list)
    steps: int = 396
    repetitions: int = 3  # min wall time is reported

    def validate(self):
        if not self.cores_list or not self.agents_list or not self.vmax_list:
            raise ValueError("SweepSpec: cores, agents and vmax lists must be non-empty")
        if any(c < 1 for c in self.cores_list):
            raise ValueError("SweepSpec: cores must be >= 1")
        if any(a < 1 for a in self.agents_list):
            raise ValueError("SweepSpec: agent counts must be >= 1")
        if any(not fp.K_MIN_VMAX <= v <= fp.K_MAX_VMAX for v in self.vmax_list):
            raise ValueError("SweepSpec: v_max must be in [1,5]")
        if self.steps < 1:
            raise ValueError("SweepSpec: steps must be >= 1")
        if self.repetitions < 1:
            raise ValueError("SweepSpec: repetitions must be >= 1")


def run_sweep(spec: SweepSpec, sc: fp.Scenario, seed: int, device: int = 0) -> List[RunRecord]:
    """run_sweep (bench.hpp:48-97): one record per (agents, v_max, cores), the minimum device
    wall time over `repetitions` identical runs; the final state must not depend on `cores`."""
    spec.validate()
    max_agents = max(spec.agents_list)
    if max_agents > sc.grid.free_cell_count():
        raise RuntimeError("run_sweep: scenario '%s' has capacity %d but the sweep asks for %d agents" %
                           (sc.name, sc.grid.free_cell_count(), max_agents))
    records = []
    for agents in spec.agents_list:
        for v_max in spec.vmax_list:
            group_hash = None
            for cores in spec.cores_list:
                params = fp.SimParams(v_max=v_max, seed=seed, steps=spec.steps)
                best = None
                final_hash = 0
                for rep in range(spec.repetitions):
                    st = fp.make_state(sc, fp.spawn_agents(sc.grid, agents, v_max, seed), device=device)
                    rs = fp.run(st, params, fp.ScheduleParams(cores))
                    if best is None or rs.wall_time_s < best.wall_time_s:
                        best = RunRecord(sc.name, agents, v_max, cores, spec.steps, rs.wall_time_s,
                                         rs.plan_time_s, rs.move_time_s, seed)
                    if rep == 0:
                        final_hash = fp.state_hash(st)
                    st.close()
                records.append(best)
                if group_hash is None:
                    group_hash = final_hash
                elif group_hash != final_hash:
                    raise RuntimeError("run_sweep: final state differs across worker counts for agents=%d, "
                                       "v_max=%d" % (agents, v_max))
    return records


@dataclass
class SpeedupRow:
    """bench.hpp:99-106."""
    scenario: str
    agents_initial: int = 0
    v_max: int = 0
    cores: int = 0
    wall_time_s: float = 0.0
    factor: float = 0.0  # wall_time(1 core) / wall_time(cores)


def speed_factor(records: Sequence[RunRecord]) -> List[SpeedupRow]:
    """speed_factor (bench.hpp:108-128): needs a 1-core baseline per (scenario, agents, v_max)."""
    baseline: Dict[Tuple[str, int, int], float] = {}
    for r in records:
        if r.cores == 1:
            baseline.setdefault((r.scenario, r.agents_initial, r.v_max), r.wall_time_s)
    rows = []
    for r in records:
        key = (r.scenario, r.agents_initial, r.v_max)
        if key not in baseline:
            raise RuntimeError("speed_factor: no 1-core baseline for scenario=%s, agents=%d, v_max=%d" %
                               (r.scenario, r.agents_initial, r.v_max))
        rows.append(SpeedupRow(r.scenario, r.agents_initial, r.v_max, r.cores, r.wall_time_s,
                               baseline[key] / r.wall_time_s))
    return rows


def speedups_to_csv(rows: Sequence[SpeedupRow]) -> str:
    """to_csv(vector<SpeedupRow>) (bench.hpp:130-149): factors with 3 decimals."""
    out = [SPEEDUP_CSV_HEADER]
    for r in rows:
        _check_csv_text(r.scenario)
        out.append("%s,%d,%d,%d,%s,%.3f" % (r.scenario, r.agents_initial, r.v_max, r.cores,
                                            _fixed6(r.wall_time_s), r.factor))
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------------- capacity
@dataclass
class CapacityResult:
    """bench.hpp:151-160."""
    capacity: int = -1  # largest N with wall_time(N) <= budget
    n_low: int = 0      # bracket: wall_time(n_low) <= budget
    n_high: int = 0     #          wall_time(n_high) > budget
    t_low_s: float = 0.0
    t_high_s: float = 0.0
    budget_s: float = 0.0
    below_start: bool = False  # budget already exceeded at the starting N
    capped: bool = False       # scenario ran out of free cells before the budget did


def realtime_capacity(wall_time_of: Callable[[int], float], budget_s: float, start_n: int = 1000,
                      max_n: int = (2 ** 63 - 1) // 2) -> CapacityResult:
    """realtime_capacity (bench.hpp:162-208): doubles N from start_n until wall_time(N) exceeds
    the budget, then interpolates linearly inside the bracket and rounds down."""
    if not budget_s > 0.0:
        raise ValueError("realtime_capacity: budget must be > 0")
    if start_n < 1:
        raise ValueError("realtime_capacity: start_n must be >= 1")
    if max_n < start_n:
        raise ValueError("realtime_capacity: max_n below start_n")
    res = CapacityResult(budget_s=budget_s)
    lo = start_n
    t_lo = wall_time_of(lo)
    if t_lo > budget_s:
        res.below_start = True
        res.n_high = lo
        res.t_high_s = t_lo
        return res
    while True:
        if lo >= max_n:
            res.capped = True
            res.capacity = lo
            res.n_low = lo
            res.t_low_s = t_lo
            return res
        hi = min(lo * 2, max_n)
        t_hi = wall_time_of(hi)
        if t_hi > budget_s:
            res.n_low, res.t_low_s, res.n_high, res.t_high_s = lo, t_lo, hi, t_hi
            # same fp64 operation order as bench.hpp:197-200
            res.capacity = int(math.floor(float(lo) + (budget_s - t_lo) * float(hi - lo) / (t_hi - t_lo)))
            return res
        lo, t_lo = hi, t_hi


def realtime_capacity_scenario(sc: fp.Scenario, v_max: int, cores: int, seed: int, budget_steps: int,
                               dt: float = 1.0, start_n: int = 1000, device: int = 0) -> CapacityResult:
    """The real-probe wrapper (bench.hpp:210-226): each probe spawns N agents and times
    budget_steps device steps, so the budget is budget_steps * dt simulated seconds."""
    params = fp.SimParams(v_max=v_max, seed=seed, steps=budget_steps, dt=dt)
    params.validate()
    if cores < 1:
        raise ValueError("run: cores must be >= 1")

    def probe(n: int) -> float:
        st = fp.make_state(sc, fp.spawn_agents(sc.grid, n, v_max, seed), device=device)
        t = fp.run(st, params, fp.ScheduleParams(cores)).wall_time_s
        st.close()
        return t

    return realtime_capacity(probe, budget_steps * dt, start_n, sc.grid.free_cell_count())


# ---------------------------------------------------------------------------------- fundamental diagram
@dataclass
class FdRecord:
    """One density-flow-speed row (bench.hpp:228-233); flow = density * mean_speed."""
    density: float = 0.0     # persons per m^2
    mean_speed: float = 0.0  # m/s
    flow: float = 0.0        # persons per meter per second


def _llround(x: float) -> int:
    """std::llround for x >= 0: halves away from zero, exact in fp64."""
    r = math.floor(x)
    return int(r) + (1 if x - r >= 0.5 else 0)


def fundamental_diagram(corridor: fp.Grid, v_max: int, densities: Sequence[float], seed: int, warmup: int = 100,
                        measure: int = 296, drive_gradient: float = K_DEFAULT_DRIVE_GRADIENT,
                        device: int = 0, k_s: float = 1.2) -> List[FdRecord]:
    """fundamental_diagram (bench.hpp:244-305) on the device: a periodic zero-exit corridor with
    the DriveX potential; after `warmup` steps the mean per-step x displacement over `measure`
    steps and all agents gives the speed at each density.  The displacement sum is the device's
    per-phase sum of segment_dx (start x, end x) over the walks -- the quantity bench.hpp:294-299
    accumulates from positions."""
    if corridor.boundary != fp.PERIODIC_X or corridor.exit_cell_count() != 0:
        raise ValueError("fundamental_diagram: corridor must be periodic-x with zero exits")
    if warmup < 0 or measure < 1:
        raise ValueError("fundamental_diagram: need warmup >= 0 and measure >= 1")
    if not drive_gradient > 0.0:
        raise ValueError("fundamental_diagram: drive gradient must be > 0")
    cell = corridor.cell_size
    free_area_m2 = corridor.free_cell_count() * cell * cell
    rho_cap = 1.0 / (cell * cell)
    field_ = None  # the corridor's (all-unreachable) exit field; DriveX never reads it
    out = []
    for rho in densities:
        if not rho >= 0.0:
            raise ValueError("fundamental_diagram: densities must be >= 0")
        n = _llround(rho * free_area_m2)
        if n > corridor.free_cell_count():
            raise RuntimeError("fundamental_diagram: density %f /m^2 exceeds the capacity 1/cell_size^2 = %f /m^2" %
                               (rho, rho_cap))
        if n < 1:
            raise ValueError("fundamental_diagram: density %f /m^2 yields zero agents on this corridor" % rho)
        params = fp.SimParams(k_s=k_s, v_max=v_max, seed=seed, steps=warmup + measure)
        if field_ is None:
            field_ = fp.compute_static_field(corridor, device)
        st = fp.SimState(corridor, field_, fp.spawn_agents(corridor, n, v_max, seed), device=device)
        st.set_potential(fp.DRIVE_X, drive_gradient)
        sched = fp.ScheduleParams(1)
        for _ in range(warmup):
            fp.step(st, params, sched)
        total_dx = 0
        for _ in range(measure):
            fp.step(st, params, sched)
            total_dx += st.last_dx
        st.close()
        density = float(n) / free_area_m2
        mean_speed = (float(total_dx) / (float(n) * float(measure))) * cell / params.dt
        out.append(FdRecord(density, mean_speed, density * mean_speed))
    return out


def fd_to_csv(records: Sequence[FdRecord]) -> str:
    """to_csv(vector<FdRecord>) (bench.hpp:307-321)."""
    out = [FD_CSV_HEADER]
    for r in records:
        out.append("%s,%s,%s" % (_fixed6(r.density), _fixed6(r.mean_speed), _fixed6(r.flow)))
    return "\n".join(out) + "\n"


def weidmann_speed(density: float) -> float:
    """weidmann_speed (bench.hpp:328-335)."""
    if density < 0.0:
        raise ValueError("weidmann_speed: density must be >= 0")
    if density >= WEIDMANN_MAX_DENSITY:
        return 0.0
    if density == 0.0:
        return WEIDMANN_FREE_SPEED
    return WEIDMANN_FREE_SPEED * (1.0 - math.exp(-WEIDMANN_GAMMA * (1.0 / density - 1.0 / WEIDMANN_MAX_DENSITY)))


@dataclass
class WeidmannRow:
    """bench.hpp:337-342."""
    density: float = 0.0
    model_speed: float = 0.0
    reference_speed: float = 0.0
    abs_error: float = 0.0


def compare_weidmann(fd: Sequence[FdRecord]) -> List[WeidmannRow]:
    """compare_weidmann (bench.hpp:344-351)."""
    rows = []
    for r in fd:
        ref = weidmann_speed(r.density)
        rows.append(WeidmannRow(r.density, r.mean_speed, ref, abs(r.mean_speed - ref)))
    return rows
