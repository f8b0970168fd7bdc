"""Command-line harness mirroring the reference's `tools/fastped.cpp` (subcommands run, sweep,
realtime, fd, speedup: same options, defaults, console lines and CSV files), on the device engine.

    python -m paper_0911_2900_b200 run --scenario plaza.txt --agents 100000 --out run.csv

Two subcommands are additions for the formats of SURVEY §8(f)3-4: `scenario` writes a built-in
workload's geometry (BASELINE configs 1-5) as a text or binary scenario file, and `trajectory`
records per-step snapshots (positions, alive bits, exit order, optional occupancy) to a FASTTRJ1
file.  Scenario files ending in `.fscb` (or starting with the FASTSCB1 magic) load as binary.

Errors follow the reference's main (`tools/fastped.cpp:210-222`): an exception prints
"fastped: <message>" to stderr and exits 1; a usage error exits 2 (argparse).
"""
from __future__ import annotations

import argparse
import sys
from typing import List, Optional, Sequence

from . import fastped as fp
from . import harness as hx
from . import scenario_io as sio


def _list(kind):
    """CLI11's `->delimiter(',')` vector options."""
    def parse(text: str):
        try:
            return [kind(t) for t in text.split(",") if t != ""]
        except ValueError:
            raise argparse.ArgumentTypeError("expected a comma-separated list: " + text) from None
    return parse


def _u64(text: str) -> int:
    v = int(text, 0)
    if not 0 <= v < 2 ** 64:
        raise argparse.ArgumentTypeError("seed must be an unsigned 64-bit integer")
    return v


def _load(path: str, device: int) -> fp.Scenario:
    try:
        with open(path, "rb") as f:
            magic = f.read(len(sio.BINARY_MAGIC))
    except OSError:
        raise RuntimeError("cannot open scenario file: " + str(path)) from None
    if magic == sio.BINARY_MAGIC:
        return sio.load_scenario_binary(path, device=device)
    return sio.load_scenario(path, device)


def _write_text(text: str, path: str):
    """write_text_file (scenario_io.hpp:179-186)."""
    try:
        with open(path, "wb") as f:
            f.write(text.encode())
    except OSError:
        raise RuntimeError("cannot write file: " + path) from None


def capacity_csv(name: str, v_max: int, cores: int, budget_steps: int, seed: int,
                 res: hx.CapacityResult) -> str:
    """capacity_csv (tools/fastped.cpp:19-39)."""
    return ("scenario,v_max,cores,budget_steps,budget_s,capacity,n_low,t_low_s,n_high,t_high_s,seed\n"
            "%s,%d,%d,%d,%.6f,%d,%d,%.6f,%d,%.6f,%d\n" % (name, v_max, cores, budget_steps, res.budget_s,
                                                          res.capacity, res.n_low, res.t_low_s, res.n_high,
                                                          res.t_high_s, seed))


# ---------------------------------------------------------------------------------- subcommands
def cmd_run(a) -> int:
    """cmd_run (tools/fastped.cpp:41-62)."""
    sc = _load(a.scenario, a.device)
    params = fp.SimParams(v_max=a.vmax, seed=a.seed, steps=a.steps)
    params.validate()
    st = fp.make_state(sc, fp.spawn_agents(sc.grid, a.agents, a.vmax, a.seed), device=a.device)
    rs = fp.run(st, params, fp.ScheduleParams(a.cores))
    st.close()
    rec = hx.RunRecord(sc.name, a.agents, a.vmax, a.cores, a.steps, rs.wall_time_s, rs.plan_time_s,
                       rs.move_time_s, a.seed)
    _write_text(hx.runs_to_csv([rec]), a.out)
    print("%s: %d agents, v_max=%d, cores=%d, %d steps" % (sc.name, a.agents, a.vmax, a.cores, a.steps))
    print("wall %.6f s (plan %.6f s, move %.6f s), exited %d, alive %d" %
          (rs.wall_time_s, rs.plan_time_s, rs.move_time_s, rs.exited, rs.alive))
    print("wrote %s" % a.out)
    return 0


def cmd_sweep(a) -> int:
    """cmd_sweep (tools/fastped.cpp:64-79)."""
    sc = _load(a.scenario, a.device)
    spec = hx.SweepSpec(cores_list=a.cores, agents_list=a.agents, vmax_list=a.vmax, steps=a.steps,
                        repetitions=a.reps)
    records = hx.run_sweep(spec, sc, a.seed, a.device)
    _write_text(hx.runs_to_csv(records), a.out)
    print("%d records -> %s" % (len(records), a.out))
    return 0


def cmd_realtime(a) -> int:
    """cmd_realtime (tools/fastped.cpp:81-106)."""
    sc = _load(a.scenario, a.device)
    res = hx.realtime_capacity_scenario(sc, a.vmax, a.cores, a.seed, a.budget_steps, a.dt, a.start_n, a.device)
    if res.below_start:
        print("capacity < %d: wall_time(%d) = %.3f s exceeds budget %.3f s" %
              (res.n_high, res.n_high, res.t_high_s, res.budget_s))
    elif res.capped:
        print("capacity >= %d (scenario ran out of free cells; wall_time(%d) = %.3f s within budget %.3f s)" %
              (res.capacity, res.n_low, res.t_low_s, res.budget_s))
    else:
        print("real-time capacity: %d agents (budget %.3f s)" % (res.capacity, res.budget_s))
        print("bracket: wall_time(%d) = %.3f s <= budget < wall_time(%d) = %.3f s" %
              (res.n_low, res.t_low_s, res.n_high, res.t_high_s))
    _write_text(capacity_csv(sc.name, a.vmax, a.cores, a.budget_steps, a.seed, res), a.out)
    print("wrote %s" % a.out)
    return 0


def cmd_fd(a) -> int:
    """cmd_fd (tools/fastped.cpp:108-124)."""
    corridor = fp.make_corridor(a.length_m, a.width_m, a.cell_size)
    fd = hx.fundamental_diagram(corridor, a.vmax, a.densities, a.seed, a.warmup, a.measure, a.drive_gradient,
                                a.device)
    print("%10s %12s %12s %14s" % ("density", "mean_speed", "flow", "weidmann_ref"))
    for row in hx.compare_weidmann(fd):
        print("%10.3f %12.3f %12.3f %14.3f" % (row.density, row.model_speed, row.density * row.model_speed,
                                              row.reference_speed))
    _write_text(hx.fd_to_csv(fd), a.out)
    print("wrote %s" % a.out)
    return 0


def cmd_speedup(a) -> int:
    """cmd_speedup (tools/fastped.cpp:126-140); host-only."""
    try:
        with open(a.in_path, "rb") as f:
            text = f.read().decode()
    except OSError:
        raise RuntimeError("cannot open csv file: " + a.in_path) from None
    rows = hx.speed_factor(hx.parse_run_csv(text))
    print("%-20s %10s %6s %6s %12s %8s" % ("scenario", "agents", "v_max", "cores", "wall_time_s", "factor"))
    for r in rows:
        print("%-20s %10d %6d %6d %12.6f %8.3f" % (r.scenario, r.agents_initial, r.v_max, r.cores, r.wall_time_s,
                                                  r.factor))
    _write_text(hx.speedups_to_csv(rows), a.out)
    print("wrote %s" % a.out)
    return 0


def cmd_scenario(a) -> int:
    """Writes a built-in workload's geometry (scenarios.py, BASELINE configs 1-5); host-only.
    Binary output (`--binary` or a `.fscb` path) can carry the device-computed field."""
    from . import scenarios
    kw = {k: v for k, v in (("width", a.width), ("height", a.height)) if v is not None}
    if kw and a.config not in ("plaza", "obstacles"):
        raise ValueError("scenario: --width/--height apply to plaza and obstacles only")
    if any(v < 3 for v in kw.values()):
        raise ValueError("scenario: width and height must be >= 3")
    wl = scenarios.build(a.config, seed=a.seed, n=0, **kw)  # geometry only: no agents
    binary = a.binary or a.out.endswith(".fscb")
    if binary:
        if a.with_field:
            sio.save_scenario_binary(fp.make_scenario(a.config, wl.grid, a.device), a.out)
        else:
            sio.save_scenario_binary(wl.grid, a.out, with_field=False)
    else:
        sio.save_scenario(wl.grid, a.out)
    print("%s: %dx%d, %d free cells, %d exit cells -> %s" % (a.config, wl.grid.width, wl.grid.height,
                                                            wl.grid.free_cell_count(), wl.grid.exit_cell_count(),
                                                            a.out))
    return 0


def cmd_trajectory(a) -> int:
    """record_trajectory (tests/acceptance.cpp:53-73) streamed to a FASTTRJ1 file."""
    sc = _load(a.scenario, a.device)
    params = fp.SimParams(v_max=a.vmax, seed=a.seed, steps=a.steps)
    params.validate()
    snaps = sio.record_trajectory(sc, a.agents, params, a.cores, a.steps, a.out, a.occupancy, a.device)
    print("%s: %d agents, %d steps, alive %d -> %s" % (sc.name, a.agents, a.steps,
                                                      int(snaps[-1].alive.sum()) if snaps else a.agents, a.out))
    return 0


# ---------------------------------------------------------------------------------- parser
def build_parser() -> argparse.ArgumentParser:
    """Options and defaults of tools/fastped.cpp:143-208."""
    ap = argparse.ArgumentParser(prog="fastped", description="fastped - grid pedestrian engine benchmark harness "
                                                             "(B200 device engine)")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p, seed=True):
        if seed:
            p.add_argument("--seed", type=_u64, default=1, help="random seed")
        p.add_argument("--device", type=int, default=0, help="CUDA device")

    p = sub.add_parser("run", help="time one simulation run")
    p.add_argument("--scenario", required=True, help="scenario file")
    p.add_argument("--agents", type=int, required=True, help="agent count")
    p.add_argument("--vmax", type=int, default=4, help="maximum speed in cells per step (1-5)")
    p.add_argument("--cores", type=int, default=1, help="planning worker count (API compatibility)")
    p.add_argument("--steps", type=int, default=396, help="simulation steps")
    p.add_argument("--out", required=True, help="output csv")
    common(p)
    p.set_defaults(fn=cmd_run)

    p = sub.add_parser("sweep", help="sweep cores x agents x vmax")
    p.add_argument("--scenario", required=True, help="scenario file")
    p.add_argument("--cores", type=_list(int), default=[1, 2, 4, 8], help="worker counts")
    p.add_argument("--agents", type=_list(int), required=True, help="agent counts")
    p.add_argument("--vmax", type=_list(int), default=[4], help="maximum speeds")
    p.add_argument("--steps", type=int, default=396, help="simulation steps per run")
    p.add_argument("--reps", type=int, default=3, help="timed repetitions per cell (min is reported)")
    p.add_argument("--out", required=True, help="output csv")
    common(p)
    p.set_defaults(fn=cmd_sweep)

    p = sub.add_parser("realtime", help="largest agent count that runs in real time")
    p.add_argument("--scenario", required=True, help="scenario file")
    p.add_argument("--vmax", type=int, default=4, help="maximum speed")
    p.add_argument("--cores", type=int, default=1, help="planning worker count")
    p.add_argument("--budget-steps", type=int, default=396, help="simulated steps = wall-clock budget in s")
    p.add_argument("--dt", type=float, default=1.0, help="seconds per step")
    p.add_argument("--start-n", type=int, default=1000, help="doubling search start")
    p.add_argument("--out", required=True, help="output csv")
    common(p)
    p.set_defaults(fn=cmd_realtime)

    p = sub.add_parser("fd", help="density/speed/flow on a periodic corridor")
    p.add_argument("--length-m", type=float, default=50.0, help="corridor length in meters")
    p.add_argument("--width-m", type=float, default=4.0, help="corridor width in meters")
    p.add_argument("--vmax", type=int, default=4, help="maximum speed")
    p.add_argument("--densities", type=_list(float), required=True, help="densities in persons/m^2")
    p.add_argument("--warmup", type=int, default=100, help="steps before measurement")
    p.add_argument("--measure", type=int, default=296, help="measured steps")
    p.add_argument("--drive-gradient", type=float, default=fp.K_DEFAULT_DRIVE_GRADIENT,
                   help="potential drop per +x cell")
    p.add_argument("--cell-size", type=float, default=0.4, help="cell size in meters")
    p.add_argument("--out", required=True, help="output csv")
    common(p)
    p.set_defaults(fn=cmd_fd)

    p = sub.add_parser("speedup", help="speed factors from a sweep csv")
    p.add_argument("--in", dest="in_path", required=True, help="sweep csv")
    p.add_argument("--out", required=True, help="output csv")
    p.set_defaults(fn=cmd_speedup)

    p = sub.add_parser("scenario", help="write a built-in workload's geometry (text, or binary .fscb)")
    p.add_argument("--config", required=True, choices=["corridor", "room", "ring", "plaza", "obstacles"])
    p.add_argument("--width", type=int, default=None, help="override the width (plaza, obstacles)")
    p.add_argument("--height", type=int, default=None, help="override the height (plaza, obstacles)")
    p.add_argument("--binary", action="store_true", help="binary FASTSCB1 output")
    p.add_argument("--with-field", action="store_true", help="binary only: store the device-computed field")
    p.add_argument("--out", required=True, help="output scenario file")
    common(p)
    p.set_defaults(fn=cmd_scenario)

    p = sub.add_parser("trajectory", help="record per-step snapshots to a FASTTRJ1 file")
    p.add_argument("--scenario", required=True, help="scenario file")
    p.add_argument("--agents", type=int, required=True, help="agent count")
    p.add_argument("--vmax", type=int, default=4, help="maximum speed")
    p.add_argument("--cores", type=int, default=1, help="planning worker count")
    p.add_argument("--steps", type=int, default=30, help="simulation steps")
    p.add_argument("--occupancy", action="store_true", help="also dump the i32 occupancy per step")
    p.add_argument("--out", required=True, help="output trajectory file")
    common(p)
    p.set_defaults(fn=cmd_trajectory)
    return ap


def main(argv: Optional[Sequence[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except Exception as e:  # tools/fastped.cpp:218-221
        print("fastped: %s" % e, file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
