#!/usr/bin/env python
"""bench.py -- agent-updates/s of the F.A.S.T. planning + motion hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config plaza] [--impl ours|reference]

A step is one simulation step (plan_phase + move_phase, engine.hpp:143-148) over the whole
roster; agent-updates = sum over steps of the alive count entering the step.
`value` is device-timed (CUDA events around fp_run's stepping loop, state resident in HBM);
`e2e` runs the same steps through the C ABI with host buffers every step (H2D of the roster,
plan+move, D2H of positions/alive), wall-clocked.  `--impl reference` times the reference's own
CPU run() (oracle/_ref, all host threads) on the same workload.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "agent-updates/sec (v_m=4, k_S=1.2)"
UNIT = "agent-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + q,
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                pass

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                for k, nm in enumerate(names):
                    if r[2 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def coverage_u(grid, x, y, v, alive):
    """U: distinct cells within Chebyshev distance v_i of some alive agent."""
    H, W = grid.height, grid.width
    mark = np.zeros((H, W), bool)
    al = alive.astype(bool)
    xs, ys, vs = x[al].astype(np.int64), y[al].astype(np.int64), v[al].astype(np.int64)
    vmax = int(vs.max()) if len(vs) else 0
    for dy in range(-vmax, vmax + 1):
        for dx in range(-vmax, vmax + 1):
            sel = np.maximum(abs(dx), abs(dy)) <= vs
            yy = ys[sel] + dy
            xx = xs[sel] + dx
            if grid.boundary == 1:
                xx %= W
                ok = (yy >= 0) & (yy < H)
            else:
                ok = (yy >= 0) & (yy < H) & (xx >= 0) & (xx < W)
            mark[yy[ok], xx[ok]] = True
    return int(mark.sum())


def plan_bytes(n_alive, U, mixed_v, drive_x):
    """Algorithmic bytes of one plan launch (SURVEY 8d B_plan)."""
    per_cell = 0.25 if drive_x else 8.25
    return n_alive * (8 + 8 + (1 if mixed_v else 0)) + U * per_cell


def build_workload(cfg, seed):
    from paper_0911_2900_b200 import scenarios
    return scenarios.build(cfg, seed=seed)


def reference_cpu(wl, field, max_steps, cores, budget_s, warmup=0):
    """The reference's own run() (oracle/_ref, unmodified headers) on this workload, from step 0:
    one calibration step, then as many more (<= max_steps - 1) as fit in ~budget_s seconds.
    `warmup` untimed steps run first on a throwaway state built from the same inputs (threads,
    page faults), so the timed run still starts at step 0.
    Returns (agent-updates/s over all timed steps, kind, cores, steps, seconds)."""
    import oracle as O
    ro = wl.roster
    if O.have_reference():
        if warmup > 0:
            w = O.RefState(wl.grid.cells, field, ro.x, ro.y, ro.v_max, ro.alive, wl.grid.boundary,
                           potential=wl.potential, drive_gradient=wl.drive_gradient)
            w.run(wl.k_s, wl.seed, warmup, cores)
            del w
        st = O.RefState(wl.grid.cells, field, ro.x, ro.y, ro.v_max, ro.alive, wl.grid.boundary,
                        potential=wl.potential, drive_gradient=wl.drive_gradient)
        upd, secs, steps = 0.0, 0.0, 0
        n0 = st.alive_count
        r = st.run(wl.k_s, wl.seed, 1, cores)
        upd, secs, steps = float(n0), r["wall_time_s"], 1
        more = int(min(max_steps - 1, max(0.0, budget_s - secs) / max(secs, 1e-9)))
        if more > 0:
            n0 = st.alive_count
            r = st.run(wl.k_s, wl.seed, more, cores)
            n1 = st.alive_count
            # alive entering each step lies between n1 and n0 (exits per step << N)
            upd += (n0 + n1) / 2.0 * more
            secs += r["wall_time_s"]
            steps += more
        return upd / secs, "reference", cores, steps, secs
    st = O.State(wl.grid.cells, field, ro.x, ro.y, ro.v_max, ro.alive, wl.grid.boundary,
                 potential=wl.potential, drive_gradient=wl.drive_gradient)
    upd, steps = 0, 0
    t0 = time.perf_counter()
    while steps < max_steps and (steps == 0 or time.perf_counter() - t0 < budget_s):
        upd += st.alive_count
        st.step_once(wl.k_s, wl.seed)
        steps += 1
    secs = time.perf_counter() - t0
    return upd / secs, "port", 1, steps, secs


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def plan_traffic(workload):
    """DRAM bytes per plan-kernel launch from the committed `ncu --set full` summary (or None)."""
    try:
        with open(os.path.join(ROOT, "profiles", "plan_kernel_ncu.json")) as f:
            p = json.load(f)
        if p.get("workload") == workload:
            return float(p["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def gpu_local_affinity(device: int):
    """Binds this process to the CPUs NVML reports as local to `device` (found by PCI bus id);
    returns the previous affinity, or None when NVML is unavailable."""
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=396)  # the reference's run length
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of reference CPU work")
    ap.add_argument("--config", default="plaza", choices=["corridor", "room", "ring", "plaza", "obstacles"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config_desc = {"workload": args.config, "seed": args.seed, "k_s": 1.2, "v_max": 4,
                   "steps_from": 0, "l2": "inputs larger than L2 (field fp64 > 126 MB)"
                   if args.config in ("plaza", "obstacles") else "L2-resident inputs; no flush"}

    if args.impl == "reference":
        if rank != 0:
            return
        wl = build_workload(args.config, args.seed)
        from paper_0911_2900_b200 import fastped as fp
        import oracle as O
        field = O.static_field(wl.grid.cells, wl.grid.boundary)
        cores = os.cpu_count() or 1
        # each "step" of this arm is the reference's own step; the run is bounded to ~60 s of work
        v, kind, c, steps_done, secs = reference_cpu(wl, field, max(1, args.steps), cores, 60.0, args.warmup)
        config_desc.update(n_agents=int(len(wl.roster)), grid=[wl.grid.width, wl.grid.height])
        sample = (f"{steps_done} of the {args.steps} steps of {args.config} from step 0 "
                  f"({secs:.1f} s, reference run() with ScheduleParams{{cores={c}}}, {cpu_model()})")
        out = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps_done,
               "warmup": args.warmup if kind == "reference" else 0, "ms_per_step": secs / steps_done * 1e3,
               "higher_is_better": True, "impl": "reference", "dtype": "f64", "data": "synthetic", "scaling": "strong",
               "vs_baseline": None, "config": config_desc,
               "cpu_baseline": {"value": v, "unit": UNIT, "cores": c, "kind": kind, "sample": sample},
               "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(out))
        return

    import torch
    import torch.distributed as dist
    from paper_0911_2900_b200 import fastped as fp

    if world > 1:
        if os.environ.get("FASTPED_DIST_BACKEND") == "gloo":  # functional check of the N>1 path on one GPU
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    wl = build_workload(args.config, args.seed)
    ro = wl.roster
    n = len(ro)
    st = fp.SimState(wl.grid, None, ro, device=local)
    if wl.potential:
        st.set_potential(wl.potential, wl.drive_gradient)
    params = fp.SimParams(k_s=wl.k_s, seed=wl.seed, steps=max(1, args.warmup))
    from paper_0911_2900_b200.dist import StripStepper, aggregate
    stepper = StripStepper(st) if world > 1 else None  # x-strip planning + replicated motion

    def strip_run(steps):
        """`steps` decomposed steps, device-timed (CUDA events; every engine call is synchronous)."""
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        upd = 0
        ev0.record()
        for _ in range(steps):
            upd += st.alive
            stepper.step(params)
        ev1.record()
        ev1.synchronize()
        return SimpleNamespace(wall_time_s=ev0.elapsed_time(ev1) * 1e-3, agent_updates=upd, steps=steps,
                               plan_time_s=None, move_time_s=None)

    # warm-up steps, then reset the roster to the initial state (untimed)
    if args.warmup > 0:
        fp.run(st, params) if stepper is None else strip_run(args.warmup)
    st.set_agents(ro.x, ro.y, ro.alive)
    st.step = 0
    # the plan kernel alone (CUDA events on its stream) on the start state; again on the end
    # state below -- the roofline uses the mean, like U (the state is re-planned by the run)
    kernel_ms0 = st.time_plan_kernel(wl.k_s, wl.seed, 20)
    c0 = st.counters()
    U0 = coverage_u(wl.grid, ro.x, ro.y, ro.v_max, ro.alive)
    params.steps = args.steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx --nvtx-include "timed/" selects these launches
        rs = fp.run(st, params) if stepper is None else strip_run(args.steps)
        torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    c1 = st.counters()
    x1, y1, a1 = st.agents()
    kernel_ms1 = st.time_plan_kernel(wl.k_s, wl.seed, 20)
    kernel_ms = 0.5 * (kernel_ms0 + kernel_ms1)
    U1 = coverage_u(wl.grid, x1, y1, ro.v_max, a1)
    # max time over ranks; the agent updates are the one simulation's (identical on every rank)
    wall, updates = aggregate(rs.wall_time_s, rs.agent_updates)
    updates /= world
    value = updates / wall

    # e2e: the C ABI with host buffers, every step H2D roster + step + D2H positions/alive.  The
    # host side runs on the GPU's NUMA-local cores and its pinned buffers are first touched there
    # (a remote socket halves the PCIe copy bandwidth); the previous affinity comes back after.
    e2e_steps = args.e2e_steps or args.steps
    saved_affinity = gpu_local_affinity(local)
    st2 = fp.SimState(wl.grid, st.field(), ro, device=local)
    if wl.potential:
        st2.set_potential(wl.potential, wl.drive_gradient)
    hx = torch.from_numpy(ro.x.copy()).pin_memory().numpy()
    hy = torch.from_numpy(ro.y.copy()).pin_memory().numpy()
    ha = torch.from_numpy(ro.alive.copy()).pin_memory().numpy()
    stepper2 = StripStepper(st2) if world > 1 else None
    # untimed e2e warm-up (a fresh context's first step allocates and instantiates its graphs:
    # 20-200 ms), then the roster goes back to the initial state
    for _ in range(max(1, args.warmup)):
        st2.set_agents(hx, hy, ha)
        fp.step(st2, params) if stepper2 is None else stepper2.step(params)
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
        upd2 += st2.alive  # counted on the device by the upload's validation pass
        fp.step(st2, params) if stepper2 is None else stepper2.step(params)
        st2.agents(out=(hx, hy, ha))  # D2H into the same pinned buffers: next step's input
    torch.cuda.synchronize()
    e2e_wall = time.perf_counter() - t0
    e2e_wall, _ = aggregate(e2e_wall, 0.0)  # slowest rank
    if saved_affinity is not None:
        os.sched_setaffinity(0, saved_affinity)
    e2e = {"value": upd2 / e2e_wall, "unit": UNIT, "h2d_bytes_per_step": n * 9, "d2h_bytes_per_step": n * 9,
           "steps": e2e_steps, "path": "fp_update_agents + fp_step + fp_get_agents (C ABI, host arrays)",
           "host_cpus": len(os.sched_getaffinity(0)) if saved_affinity is None else "gpu-local NUMA node"}

    if rank != 0:
        return
    peak, peak_kind = peaks()
    mixed = bool((ro.v_max != ro.v_max[0]).any()) if n else False
    U = 0.5 * (U0 + U1)
    nalive_avg = rs.agent_updates / max(rs.steps, 1)
    bytes_per_launch = plan_bytes(nalive_avg, U, mixed, wl.potential == fp.DRIVE_X)
    plan_launch_s = kernel_ms * 1e-3
    achieved = bytes_per_launch / plan_launch_s / 1e9
    roof = {"kernel": "plan_tile_kernel", "bound": "hbm", "achieved": achieved, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": plan_traffic(args.config),
            "bytes_per_launch": bytes_per_launch, "U_cells": U, "plan_ms_per_launch": plan_launch_s * 1e3,
            "plan_ms_start_end": [kernel_ms0, kernel_ms1], "U_start_end": [U0, U1],
            "plan_share_of_step": plan_launch_s * rs.steps / rs.wall_time_s,
            "layout_bytes_per_launch": nalive_avg * (8 + 8 + (1 if mixed else 0)) + wl.grid.width * wl.grid.height * 4.25,
            "layout_note": "this kernel streams 4 B weight-plane words + 1 occupancy bit per cell of every non-empty tile (+halo)"}

    cpu = None
    if not args.no_cpu_baseline:
        field = st.field()
        cores = os.cpu_count() or 1
        # bounded sample: one calibration step, then steps up to ~cpu_budget seconds of CPU work
        v, kind, c, steps_done, secs = reference_cpu(wl, field, args.steps, cores, args.cpu_budget)
        cpu = {"value": v, "unit": UNIT, "cores": c, "kind": kind,
               "sample": f"first {steps_done} of {args.steps} steps of {args.config} ({n} agents), {secs:.1f} s, "
                         f"reference run() on {c} threads, {cpu_model()}"}

    # real-time capacity (bench.hpp:165-226 rule, 1 step = 1 simulated s): the agent count whose
    # 396 steps take 396 s, extrapolated linearly from this run and capped at the free cells
    free_cells = int((wl.grid.cells == 0).sum())
    sec_per_step = wall / max(rs.steps, 1)
    cap_est = nalive_avg * world / max(sec_per_step, 1e-12)
    capacity = {"value": int(min(cap_est, free_cells)), "capped": bool(cap_est >= free_cells),
                "extrapolated_from_n": int(n), "free_cells": free_cells,
                "method": "linear in N from this run's ms_per_step; geometry fixed"}

    config_desc.update(n_agents=n, grid=[wl.grid.width, wl.grid.height], mixed_v=mixed)
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": wall / max(rs.steps, 1) * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": config_desc,
           "parallelism": f"x-strips{world} plan + NCCL all-reduce + replicated motion" if world > 1 else "single",
           "phases_ms": ({"plan": rs.plan_time_s * 1e3, "move": rs.move_time_s * 1e3, "total": rs.wall_time_s * 1e3}
                         if stepper is None else {"total": rs.wall_time_s * 1e3}),
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
           "realtime_capacity": capacity,
           "gpu_launches": int(c1["kernel_launches"] - c0["kernel_launches"]),
           "motion_rounds_per_step": (c1["motion_rounds"] - c0["motion_rounds"]) / max(rs.steps, 1),
           "plan_fallbacks_per_step": (c1["plan_fallbacks"] - c0["plan_fallbacks"]) / max(rs.steps, 1)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
