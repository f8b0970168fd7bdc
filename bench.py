#!/usr/bin/env python
"""bench.py -- agent-updates/s of the F.A.S.T. planning + motion hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config plaza] [--impl ours|reference]
                    [--capacity] [--v-sweep] [--fd]

A step is one simulation step (plan_phase + move_phase, engine.hpp:143-148) over the whole
roster; agent-updates = sum over steps of the alive count entering the step.

ours (default): `value` = device-timed agent-updates/s of K steps from step 0 (CUDA events on the
engine's stream around fp_run's loop, state resident in HBM, inputs larger than L2);
`full_run` = the same for the reference's whole 396-step run; `e2e` = the same steps through the
C ABI with host buffers every step (H2D roster, plan + move, D2H positions/alive), wall-clocked;
`roofline` = the plan kernel's algorithmic bytes (SURVEY 8d B_plan) / its CUDA-event launch
time on the start state and on the end state of the 396-step run; `traffic` = ncu DRAM bytes per
launch captured on those same two states (`--plan-state start|end`, profiles/plan_kernel_ncu.json);
`cpu_baseline` = the reference's own run() (oracle/_ref) on the host's physical cores.

--impl reference: the reference's own run() (oracle/_ref, the unmodified headers) on this host's
physical cores (tests/acceptance.cpp:25-44 counting), plus a cores=1 run; workload built by the
checker-side generators (oracle/configs.py) and the reference's own spawn_agents and
compute_static_field -- nothing of the product package is imported on that path.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-updates/sec (v_m=4, k_S=1.2)"
UNIT = "agent-updates/s"
RUN_STEPS = 396  # the reference's run length

# Workload metadata both arms report identically (BASELINE.json configs[0..4]).
CONFIG_META = {
    "corridor": dict(grid=[250, 50], n_agents=2000, v_max=4, mixed_v=False, potential="ExitDistance"),
    "room": dict(grid=[1000, 1000], n_agents=40000, v_max=4, mixed_v=False, potential="ExitDistance"),
    "ring": dict(grid=[4000, 200], n_agents=182000, v_max=4, mixed_v=False, potential="DriveX g=1",
                 boundary="periodic-x"),
    "plaza": dict(grid=[20000, 5000], n_agents=1000000, v_max=4, mixed_v=False, potential="ExitDistance"),
    "obstacles": dict(grid=[40000, 10000], n_agents=10000000, v_max="2..5", mixed_v=True,
                      potential="ExitDistance"),
}


def config_desc(args):
    d = {"workload": args.config, "seed": args.seed, "k_s": 1.2, "steps_from": 0}
    d.update(CONFIG_META[args.config])
    if getattr(args, "v", None):
        d["v_max"] = args.v
    d["l2"] = ("inputs larger than L2 (fp64 field / weight plane > 126 MB)" if args.config in ("plaza", "obstacles")
               else "L2-resident inputs (< 126 MB); no flush -- SURVEY 8d reports configs 1-3 as latency")
    return d


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """SM clocks and throttle reasons sampled with NVML every ~2 ms during a timed region
    (B200_PROFILING.md clocks line); a thread started before the region, so even a short
    region gets samples."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index=0):
        self.index, self.rows, self.h, self.on = index, [], None, False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_sm = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.h = None

    def _loop(self):
        nv = self.nv
        while self.on:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.rows.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.h is not None:
            self.on = True
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
            time.sleep(0.005)  # first sample lands before the region starts
        return self

    def __exit__(self, *a):
        if self.on:
            self.on = False
            self.t.join(1.0)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [r[0] for r in self.rows]
        reasons = sorted({k for _, bits in self.rows for k, m in self.REASONS.items() if bits & m})
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": float(min(sm)), "sm_max_mhz": float(self.max_sm),
                "reasons": reasons, "samples": len(sm), "source": "NVML every ~2 ms"}


def coverage_u(cells, boundary, x, y, v, alive):
    """U: distinct cells within Chebyshev distance v_i of some alive agent."""
    H, W = cells.shape
    mark = np.zeros((H, W), bool)
    al = alive.astype(bool)
    xs, ys, vs = x[al].astype(np.int64), y[al].astype(np.int64), v[al].astype(np.int64)
    vmax = int(vs.max()) if len(vs) else 0
    for dy in range(-vmax, vmax + 1):
        for dx in range(-vmax, vmax + 1):
            sel = np.maximum(abs(dx), abs(dy)) <= vs
            yy = ys[sel] + dy
            xx = xs[sel] + dx
            if boundary == 1:
                xx %= W
                ok = (yy >= 0) & (yy < H)
            else:
                ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
            mark[yy[ok], xx[ok]] = True
    return int(mark.sum())


def plan_bytes(n_alive, U, mixed_v, drive_x):
    """Algorithmic bytes of one plan launch (SURVEY 8d B_plan): per alive agent 8 B position read
    + 8 B desired write (+1 B v_max when mixed); per covered cell 8 B fp64 S + 1/8 B occupancy +
    1/8 B wall (DriveX reads no S: 1/4 B)."""
    per_cell = 0.25 if drive_x else 8.25
    return n_alive * (8 + 8 + (1 if mixed_v else 0)) + U * per_cell


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------------- reference arm (CPU)
def reference_run(cfg, cores, max_steps, budget_s, warmup=0, field=None):
    """The reference's own run() (oracle/_ref) on `cfg` from step 0, one run() call per step so
    the alive count entering every step is exact; stops after max_steps or ~budget_s seconds of
    timed stepping.  `warmup` untimed steps first run on a throwaway state (threads, page
    faults).  Returns dict(value, steps, seconds, plan_s, move_s)."""
    import oracle as O
    if field is None:
        field = O.ref_static_field(cfg.cells, cfg.boundary)  # the reference's compute_static_field
    if warmup > 0:
        w = O.RefState(cfg.cells, field, cfg.x, cfg.y, cfg.v, boundary=cfg.boundary, potential=cfg.potential,
                       drive_gradient=cfg.drive_gradient)
        w.run(cfg.k_s, cfg.seed, warmup, cores)
        del w
    st = O.RefState(cfg.cells, field, cfg.x, cfg.y, cfg.v, boundary=cfg.boundary, potential=cfg.potential,
                    drive_gradient=cfg.drive_gradient)
    upd, secs, plan, move, steps = 0, 0.0, 0.0, 0.0, 0
    while steps < max_steps and (steps == 0 or secs < budget_s):
        upd += st.alive_count
        r = st.run(cfg.k_s, cfg.seed, 1, cores)
        secs += r["wall_time_s"]
        plan += r["plan_time_s"]
        move += r["move_time_s"]
        steps += 1
    return dict(value=upd / secs, steps=steps, seconds=secs, plan_s=plan, move_s=move, updates=upd)


def reference_arm(args):
    import oracle as O
    import oracle.configs as OC
    if not O.have_reference():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference headers absent)"}))
        return
    kw = {"v": args.v} if args.v and args.config in ("corridor", "room", "plaza") else {}
    cfg = OC.build(args.config, seed=args.seed, **kw)
    cores = O.physical_core_count()
    field = O.ref_static_field(cfg.cells, cfg.boundary)
    r = reference_run(cfg, cores, max(1, args.steps), args.ref_budget, args.warmup, field)
    r1 = reference_run(cfg, 1, max(1, args.steps), args.ref_budget_1core, 0, field)
    sample = (f"first {r['steps']} of the {args.steps} steps of {args.config} from step 0 "
              f"({r['seconds']:.1f} s timed), reference run() with ScheduleParams{{cores={cores}}} "
              f"(physical cores, acceptance.cpp:25-44 counting; {os.cpu_count()} logical), {cpu_model()}")
    out = {"metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": r["steps"],
           "warmup": args.warmup, "ms_per_step": r["seconds"] / r["steps"] * 1e3, "higher_is_better": True,
           "impl": "reference", "dtype": "f64", "data": "synthetic", "scaling": "weak", "vs_baseline": None,
           "config": config_desc(args),
           "phases_ms": {"plan": r["plan_s"] * 1e3, "move": r["move_s"] * 1e3, "total": r["seconds"] * 1e3},
           "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
           "cores1": {"value": r1["value"], "steps": r1["steps"], "seconds": r1["seconds"],
                      "speed_factor": r["value"] / r1["value"]},
           "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "workload_source": "oracle/configs.py + the reference's spawn_agents / compute_static_field (oracle/_ref)"}
    print(json.dumps(out))


# --------------------------------------------------------------------------------- our arm
def build_workload(args):
    from paper_0911_2900_b200 import scenarios
    kw = {"v": args.v} if args.v and args.config in ("corridor", "room", "plaza") else {}
    return scenarios.build(args.config, seed=args.seed, **kw)


def new_state(fp, wl, device, field=None):
    st = fp.SimState(wl.grid, field, wl.roster, device=device)
    if wl.potential:
        st.set_potential(wl.potential, wl.drive_gradient)
    return st


def plan_traffic(workload, state):
    """ncu DRAM bytes per plan-kernel launch on the given state (profiles/plan_kernel_ncu.json,
    captured with `bench.py --plan-state start|end` under ncu --set full), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "plan_kernel_ncu.json")) as f:
            p = json.load(f)
        e = p.get(workload, {}).get(state)
        return float(e["dram_bytes_per_launch"]) if e else None
    except Exception:
        return None


def gpu_local_affinity(device: int):
    """Binds this process to the CPUs NVML reports as local to `device`; returns the previous
    affinity, or None when NVML is unavailable."""
    try:
        import pynvml
        import torch
        props = torch.cuda.get_device_properties(device)
        bus = "%08x:%02x:%02x.0" % (props.pci_domain_id, props.pci_bus_id, props.pci_device_id)
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        saved = os.sched_getaffinity(0)
        pynvml.nvmlDeviceSetCpuAffinity(h)
        return saved
    except Exception:
        return None


def plan_state_mode(args, fp, wl, device):
    """--plan-state start|end: puts the engine in the bench's start state (step 0) or end state
    (after the 396-step run) and launches the plan kernel 3 times -- the launches ncu captures
    for `traffic`."""
    st = new_state(fp, wl, device)
    if args.plan_state == "end":
        fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=RUN_STEPS))
    ms = st.time_plan_kernel(wl.k_s, wl.seed, 3)
    print(json.dumps({"plan_state": args.plan_state, "workload": args.config, "plan_ms": ms, "alive": st.alive}))


def capacity_probe(args, fp, wl, device, field):
    """realtime_capacity (bench.hpp:165-226) measured on the device: N doubles from 1000, each
    probe spawns N agents (spawn_agents, seed) and times `capacity_steps` device steps; the budget
    is capacity_steps simulated seconds (1 step = 1 s); capped at the free-cell count."""
    from paper_0911_2900_b200 import harness
    probes = []
    steps = args.capacity_steps

    def probe(n):
        ro = fp.spawn_agents(wl.grid, n, int(wl.roster.v_max[0]), wl.seed)
        if args.config == "obstacles":
            from paper_0911_2900_b200.scenarios import rng_u64_np
            ro.v_max = (2 + (rng_u64_np(wl.seed, np.arange(n, dtype=np.uint64), 0, 1) % np.uint64(4))).astype(np.int32)
        st = fp.SimState(wl.grid, field, ro, device=device)
        if wl.potential:
            st.set_potential(wl.potential, wl.drive_gradient)
        r = fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=steps))
        st.close()
        probes.append({"n": int(n), "wall_s": r.wall_time_s, "ms_per_step": r.wall_time_s / steps * 1e3})
        return r.wall_time_s

    t0 = time.time()
    res = harness.realtime_capacity(probe, float(steps), 1000, wl.grid.free_cell_count())
    return {"value": int(res.capacity), "capped": bool(res.capped), "n_low": int(res.n_low),
            "t_low_s": res.t_low_s, "n_high": int(res.n_high), "t_high_s": res.t_high_s,
            "budget_s": float(steps), "steps_per_probe": steps, "free_cells": int(wl.grid.free_cell_count()),
            "probes": probes, "probe_wall_s": time.time() - t0,
            "method": "bench.hpp:165-226 rule, every probe a measured device run() of steps_per_probe steps "
                      "from step 0 (1 step = 1 simulated second)"}


def ours_arm(args):
    import torch
    import torch.distributed as dist
    from paper_0911_2900_b200 import fastped as fp
    from paper_0911_2900_b200.dist import aggregate

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        if os.environ.get("FASTPED_DIST_BACKEND") == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    wl = build_workload(args)
    if args.plan_state:
        return plan_state_mode(args, fp, wl, local)
    ro = wl.roster
    n = len(ro)
    if world > 1:
        # one simulation over `world` x-strips, one GPU each (strip.cu): the ranks
        # exchange the band-connected walks once per step (NCCL allgatherv over NVLink)
        from paper_0911_2900_b200.dist import strip_rank
        transport = os.environ.get("FASTPED_STRIP_TRANSPORT", "nccl")

        def make_state(field=None):
            s_ = strip_rank(wl.grid, field, ro, local, transport=transport)
            if wl.potential:
                s_.set_potential(wl.potential, wl.drive_gradient)
            return s_
    else:
        def make_state(field=None):
            return new_state(fp, wl, local, field)
    st = make_state()
    field = st.field()
    params = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=max(1, args.warmup))

    if args.warmup > 0:
        fp.run(st, params)
    st.set_agents(ro.x, ro.y, ro.alive)
    st.step = 0
    kernel_ms0 = st.time_plan_kernel(wl.k_s, wl.seed, 20)
    c0 = st.counters()
    params.steps = args.steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        rs = fp.run(st, params)
    torch.cuda.synchronize()
    run_dx = st.run_dx
    c1 = st.counters()
    # max over ranks of the device time; the agent-updates are the simulation's (global on every
    # strip rank, so rank 0's count is the job's)
    wall, _ = aggregate(rs.wall_time_s, 0.0)
    updates = float(rs.agent_updates)
    value = updates / wall

    # the whole 396-step run from step 0 (the reference's run length), when K is shorter
    full = None
    if args.steps != RUN_STEPS:
        st.set_agents(ro.x, ro.y, ro.alive)
        st.step = 0
        with Clocks(local) as clk_full:
            rf = fp.run(st, fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=RUN_STEPS))
        wf, _ = aggregate(rf.wall_time_s, 0.0)
        uf = float(rf.agent_updates)
        full = {"steps": RUN_STEPS, "value": uf / wf, "ms_per_step": wf / RUN_STEPS * 1e3,
                "phases_ms": {"plan": rf.plan_time_s * 1e3, "move": rf.move_time_s * 1e3},
                "clocks": clk_full.summary()}
        end_steps = RUN_STEPS
    else:
        end_steps = args.steps
    # end state of the 396-step run (if the timed run was not it, `st` now holds it)
    x1, y1, a1 = st.agents()
    x1, y1, a1 = x1.copy(), y1.copy(), a1.copy()
    own1 = st.owned().astype(np.uint8) if world > 1 else None
    kernel_ms1 = st.time_plan_kernel(wl.k_s, wl.seed, 20)

    # e2e: the C ABI with host buffers, every step H2D roster + step + D2H positions/alive
    e2e_steps = args.e2e_steps or args.steps
    saved_affinity = gpu_local_affinity(local)
    st2 = make_state(field)
    hx = torch.from_numpy(ro.x.copy()).pin_memory().numpy()
    hy = torch.from_numpy(ro.y.copy()).pin_memory().numpy()
    ha = torch.from_numpy(ro.alive.copy()).pin_memory().numpy()
    p1 = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=1)
    for _ in range(max(1, args.warmup)):  # a fresh context's first steps build its graphs
        st2.set_agents(hx, hy, ha)
        fp.step(st2, p1)
        st2.agents(out=(hx, hy, ha))
    hx[:], hy[:], ha[:] = ro.x, ro.y, ro.alive
    st2.step = 0
    upd2 = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        st2.set_agents(hx, hy, ha)
        upd2 += st2.alive
        fp.step(st2, p1)
        st2.agents(out=(hx, hy, ha))
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - t0
    e2e_wall, _ = aggregate(e2e_wall, 0.0)
    if saved_affinity is not None:
        os.sched_setaffinity(0, saved_affinity)
    st2.close()
    e2e = {"value": upd2 / e2e_wall, "unit": UNIT, "h2d_bytes_per_step": n * 9, "d2h_bytes_per_step": n * 9,
           "steps": e2e_steps, "path": "fp_update_agents + fp_step + fp_get_agents (C ABI, pinned host arrays)"}

    capacity = None
    if args.capacity and world == 1:
        capacity = capacity_probe(args, fp, wl, local, field)

    if rank != 0:
        return
    peak, peak_kind = peaks()
    mixed = bool((ro.v_max != ro.v_max[0]).any()) if n else False
    drive = wl.potential == fp.DRIVE_X
    if world > 1:  # rank 0's strip: the agents it plans
        a0m = ro.alive & (ro.x >= st.x_lo) & (ro.x < st.x_hi)
        a1 = a1 & own1
    else:
        a0m = ro.alive
    U0 = coverage_u(wl.grid.cells, wl.grid.boundary, ro.x, ro.y, ro.v_max, a0m)
    U1 = coverage_u(wl.grid.cells, wl.grid.boundary, x1, y1, ro.v_max, a1)
    b0 = plan_bytes(int(a0m.sum()), U0, mixed, drive)
    b1 = plan_bytes(int(a1.sum()), U1, mixed, drive)
    a_start, a_end = b0 / (kernel_ms0 * 1e-3) / 1e9, b1 / (kernel_ms1 * 1e-3) / 1e9
    achieved = 0.5 * (a_start + a_end)
    t0_, t1_ = plan_traffic(args.config, "start"), plan_traffic(args.config, "end")
    roof = {"kernel": "plan_stream_kernel", "bound": "hbm", "achieved": achieved, "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": achieved / peak,
            "traffic": (0.5 * (t0_ + t1_)) if (t0_ and t1_) else None,
            "bytes_per_launch": 0.5 * (b0 + b1),
            "states": {"start": {"step": 0, "alive": int(ro.alive.sum()), "U_cells": U0, "bytes": b0,
                                 "plan_ms": kernel_ms0, "achieved_gbs": a_start, "frac": a_start / peak,
                                 "ncu_dram_bytes": t0_},
                       "end": {"step": end_steps, "alive": int(a1.sum()), "U_cells": U1, "bytes": b1,
                               "plan_ms": kernel_ms1, "achieved_gbs": a_end, "frac": a_end / peak,
                               "ncu_dram_bytes": t1_}},
            "how": "B_plan(state) / CUDA-event launch time (20 launches) on the start state and on the end state "
                   "of the 396-step run; achieved = mean of the two; traffic = mean ncu DRAM bytes on the same states",
            "plan_share_of_step": rs.plan_time_s / rs.wall_time_s if rs.wall_time_s else None}

    cpu = None
    if not args.no_cpu_baseline:
        import oracle as O
        import oracle.configs as OC
        if O.have_reference():
            kw = {"v": args.v} if args.v and args.config in ("corridor", "room", "plaza") else {}
            cfg = OC.build(args.config, seed=args.seed, **kw)
            cores = O.physical_core_count()
            r = reference_run(cfg, cores, args.steps, args.cpu_budget)
            cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": f"first {r['steps']} of {args.steps} steps of {args.config} ({n} agents), "
                             f"{r['seconds']:.1f} s, reference run() on {cores} physical cores, {cpu_model()}"}

    fd = None
    if wl.potential == fp.DRIVE_X:  # fundamental-diagram sampling (bench.hpp:244-305), fused in the motion
        free_area = float(wl.grid.free_cell_count()) * wl.grid.cell_size ** 2
        speed = run_dx * wl.grid.cell_size / max(float(rs.agent_updates), 1.0)  # dt = 1 s
        fd = {"density_per_m2": n / free_area, "mean_speed_mps": speed, "flow_per_m_s": n / free_area * speed,
              "note": "sum of segment_dx per step, reduced in the motion kernel (timed run)"}
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": wall / max(rs.steps, 1) * 1e3, "higher_is_better": True,
           "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_desc(args),
           "parallelism": (f"x-strips{world}: one simulation, strip per GPU, band-connected walks exchanged "
                           f"once per step ({os.environ.get('FASTPED_STRIP_TRANSPORT', 'nccl')})") if world > 1
                          else "single",
           "phases_ms": {"plan": rs.plan_time_s * 1e3, "move": rs.move_time_s * 1e3, "total": rs.wall_time_s * 1e3},
           "full_run": full, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
           "realtime_capacity": capacity, "fundamental_diagram": fd,
           "gpu_launches": int(c1["kernel_launches"] - c0["kernel_launches"]),
           "motion_rounds_per_step": (c1["motion_rounds"] - c0["motion_rounds"]) / max(rs.steps, 1),
           "plan_fallbacks_per_step": (c1["plan_fallbacks"] - c0["plan_fallbacks"]) / max(rs.steps, 1)}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=RUN_STEPS)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="plaza", choices=list(CONFIG_META))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--v", type=int, default=None, help="uniform v_max override (corridor / room / plaza)")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of reference CPU work (ours arm)")
    ap.add_argument("--ref-budget", type=float, default=60.0, help="seconds of reference work (reference arm)")
    ap.add_argument("--ref-budget-1core", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--capacity", action="store_true", help="measure realtime_capacity (bench.hpp:165-226)")
    ap.add_argument("--capacity-steps", type=int, default=RUN_STEPS)
    ap.add_argument("--plan-state", choices=["start", "end"], default=None)
    args = ap.parse_args()
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        return reference_arm(args)
    return ours_arm(args)


if __name__ == "__main__":
    main()
