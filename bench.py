#!/usr/bin/env python
"""Benchmark: grid-point RK-stage updates/s of the fused WENO5 RHS + SSP-RK3
stage (BASELINE.json metric) on B200, weak-scaled over radial slabs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--mode mixed|f64] [--nrho 65536] [--ntheta 512]

Workload (config.workload): BASELINE configs[4] shape, 65536 x 512 grid
points PER GPU (radial slabs of a (65536 N) x 512 grid), extremal-Kerr
s=-2 m=2 sign structure, WENO5, SSP-RK3, mixed precision (fp32 WENO
weights, fp64 state) as the headline and fp64 beside it.  Inputs are larger
than L2 (state 1.07 GB per register, coefficients 2.4 GB), so no explicit
L2 flush is needed between steps.  Coefficients are the reference's own
extremal-Kerr planes, assembled on the GPU by hwg_assemble_coefficients
(the reference's generated wave_op_coeffs kernels in double-double,
paper_2010_04760_b200/planes.py; untimed setup, ~3.5 min of serial host
work in the reference); the initial state is a Gaussian pulse.

One JSON line on rank 0.  See DESIGN.md §5 for the roofline bookkeeping.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "grid-point RK-stage updates/s (WENO5 mixed & fp64) at 1/2/4/8 B200, % HBM roofline"
UNIT = "stage-updates/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self):
        self.marks.append(time.time())

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t0, t1 = (self.marks + [0, 0])[:2] if len(self.marks) >= 2 else (0, 1e30)
        rows = [r for t, r in self.rows if t0 <= t <= t1] or [r for _, r in self.rows]
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 4 + i and r[4 + i].lower().startswith("active")})
        pw = [float(r[2]) for r in rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_median": float(np.median(pw)) if pw else None,
                "samples": len(rows)}


_T0 = time.time()


def log(msg):
    """Progress on stderr (the driver parses stdout's JSON line only)."""
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# --------------------------------------------------------------------- reference arm
def host_info():
    """CPU facts for the baseline record: usable cores and the load before the run."""
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count() or 1
    try:
        load = os.getloadavg()[0]
    except Exception:
        load = None
    return usable, load


def reference_rates(nrho, ntheta, modes=("mixed",), warm=1, steps=3, workers=None):
    """The UNMODIFIED reference (oracle/_ref) on the host cores, on the GPU
    arm's own grid and physics (C5 shape: extremal Kerr a=1, s=-2, m=2,
    WENO5, SSP-RK3, hook off, default FP environment): make_grid +
    assemble_coefficients (on theta-row sub-grids from `workers` threads,
    bitwise the serial result; untimed) + initial_data (untimed), then ONE
    advance_steps call over warm + steps steps with a timestamp hook, as the
    reference's bench-scaling harness does (proj/tools/main.cpp:168-221).
    The first `warm` steps (they include the stepper's scratch allocation)
    are excluded; the rate is P * 3 * steps / (sum of the timed steps).
    Workers: all usable cores but one, so the pool's per-phase barriers do
    not wait on a thread descheduled by the box's own processes."""
    import oracle as O
    usable, load = host_info()
    workers = workers or max(1, usable - 1)
    phys = O.Physics(a=1.0, spin=-2, mmode=2, ell=2, center=1.0, width=0.22)
    out = {}
    for mode in modes:
        t0 = time.perf_counter()
        ref = O.RefSolver(phys, nrho, ntheta, mode=mode, workers=workers)
        u, lo = ref.initial_data()
        setup = time.perf_counter() - t0
        dt = ref.select_dt("ssprk33")
        (u, lo), st, per = ref.advance_timed(u, lo, dt, 0, warm + steps)
        if st["blew_up"]:
            raise RuntimeError(f"reference {mode}: blew up")
        timed = per[warm:]
        wall = float(timed.sum())
        out[mode] = {"value": nrho * ntheta * 3 * steps / wall, "unit": UNIT, "steps": steps,
                     "warm_steps": warm, "wall_s": wall, "per_step_s": [float(x) for x in timed],
                     "warm_step_s": [float(x) for x in per[:warm]], "setup_s": setup}
        del ref, u, lo
    return out, workers, usable, load


def ref_sample(nrho, ntheta, mode, r, workers, usable):
    return (f"{nrho}x{ntheta} grid (the GPU arm's per-GPU workload), C5 physics (a=1, s=-2, "
            f"m=2), reference {mode} ({'DD state + fp64 weights' if mode == 'mixed' else 'DD'}), "
            f"weno5, ssprk33, {r['steps']} steps timed after {r['warm_steps']} warm-up in one "
            f"advance_steps call, {workers} pool workers of {usable} usable cores, "
            f"{r['wall_s']:.1f} s")


def cpu_reference_rate(nrho, ntheta, steps=3):
    """The GPU arm's cpu_baseline: the reference arm's measurement (mixed,
    same grid, same procedure), or the C restatement when oracle/_ref is absent."""
    import oracle as O
    if O.ref_available():
        rr, workers, usable, load = reference_rates(nrho, ntheta, ("mixed",), 2, steps)
        r = rr["mixed"]
        return {"value": r["value"], "unit": UNIT, "cores": workers, "kind": "reference",
                "sample": ref_sample(nrho, ntheta, "mixed", r, workers, usable),
                "per_step_s": r["per_step_s"], "loadavg_before": load}
    # fall back to the C restatement (single thread) on a bounded sample
    from paper_2010_04760_b200 import synthetic
    n, nt = 1024, 512
    prob = synthetic.problem(n, nt)
    orc = O.OracleSolver(n, nt, prob["drho"], prob["dtheta"], prob["parity"],
                         prob["coef"], prob["cotth"], "weno5", "mixed")
    u = synthetic.initial_state(prob)
    t0 = time.time()
    k = 0
    while time.time() - t0 < 10.0:
        u, _ = orc.advance(u, synthetic.select_dt(prob), k, k + 1)
        k += 1
    wall = time.time() - t0
    return {"value": n * nt * 3 * k / wall, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{n}x{nt} synthetic, C restatement, {k} steps"}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref,
    the unmodified library) on the host cores, on the GPU arm's config
    (args.nrho x args.ntheta, C5 physics, WENO5, SSP-RK3), both reference
    modes: mixed (the GPU mixed tier's parity reference and
    the line's value) and full.  A reference step at this size takes seconds,
    so the timed steps are capped (min(K, 3) after min(W, 2) warm-up) to keep
    the run within a few minutes; the per-step times are reported."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle as O
    nrho, ntheta = args.nrho, args.ntheta
    K, W = min(args.steps, args.ref_steps), min(args.warmup, 2)
    if not O.ref_available():
        c = cpu_reference_rate(nrho, ntheta)
        modes, v, kind, cores, sample = {}, c["value"], c["kind"], c["cores"], c["sample"]
        wall = 0.0
    else:
        modes, workers, usable, load = reference_rates(nrho, ntheta, ("mixed", "full"), W, K)
        r = modes["mixed"]
        v, kind, cores, wall = r["value"], "reference", workers, r["wall_s"]
        sample = ref_sample(nrho, ntheta, "mixed", r, workers, usable)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": K, "steps_requested": args.steps, "warmup": W,
            "ms_per_step": 1000 * wall / max(K, 1),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "dd state, fp64 weights",
            "data": "the reference's own make_grid + assemble_coefficients planes (C5 physics) "
                    "and initial_data (ell=2 Gaussian)",
            "config": {"workload": f"C5 shape {nrho}x{ntheta} per GPU, C5 physics (a=1, s=-2, "
                                   f"m=2), WENO5, SSP-RK3 (the B200 arm's workload)",
                       "scheme": "weno5", "stepper": "ssprk33", "mode": "reference mixed",
                       "same_config": True},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample},
            "modes": modes,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if "full" in modes:
        line["mixed_vs_full_speedup"] = modes["mixed"]["value"] / modes["full"]["value"]
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- B200 arm
def make_runner(args, g, mode, rank, world, dist):
    """Slab transport for N > 1: the fused halo push over NVLink peer memory
    (slabs.PeerSlab) for the fp64 / mixed tiers, NCCL point-to-point
    otherwise (or with --halo nccl)."""
    from paper_2010_04760_b200 import slabs
    if world > 1 and args.halo == "peer" and not mode.startswith("dd"):
        import torch
        r = slabs.PeerSlab(g, rank, world, "weno5")
        t = torch.tensor([0 if r.error else 1], device=f"cuda:{torch.cuda.current_device()}",
                         dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 1:
            r.prime()
            return r, "peer"
        print(f"[bench rank {rank}] no peer mappings ({r.error}); NCCL halos", file=sys.stderr)
        if r.error is None:
            g.set_peers(None, None)
    # NCCL P2P with the exchange overlapped with the interior rows (fast tiers)
    overlap = not mode.startswith("dd")
    return (slabs.DistSlab(g, rank, world, "weno5", overlap=overlap),
            ("nccl-overlap" if overlap else "nccl") if world > 1 else "none")


def time_mode(args, mode, prob, world, rank, dev, torch, dist, steps=None, warmup=None,
              stepper="ssprk33"):
    from paper_2010_04760_b200 import hwgpu, slabs, synthetic
    spec = hwgpu.SchemeSpec("weno5", mode)
    K = steps or args.steps
    W = args.warmup if warmup is None else warmup
    g = hwgpu.GpuEvolution(prob["nrho"], prob["ntheta"], prob["drho"], prob["dtheta"],
                           prob["parity"], prob["coef"], prob["cotth"], spec, device=dev,
                           rho_offset=prob["rho_offset"], nrho_global=prob["nrho_global"],
                           coef_ld=prob["nrho"], coef_row0=0)
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)
    u0 = synthetic.initial_state(prob)
    g.set_state(u0)
    dt = synthetic.select_dt(prob, stepper)
    ns = 3 if stepper == "ssprk33" else 10
    runner, halo = make_runner(args, g, mode, rank, world, dist)
    P = prob["nrho"] * prob["ntheta"]
    for q in range(W):
        runner.step(stepper, dt, q)
    torch.cuda.synchronize()
    if halo == "peer":
        # all ranks agree the fused halo push works here, else fall back to NCCL
        ok = 1
        try:
            g.status()
        except hwgpu.HwgError as e:
            print(f"[bench rank {rank}] fused halo push failed ({e}); NCCL halos", file=sys.stderr)
            ok = 0
        t = torch.tensor([ok], device=f"cuda:{dev}", dtype=torch.int32)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        if int(t.item()) == 0:
            g.set_peers(None, None)
            g.status(clear=True)
            g.set_state(u0)
            runner, halo = slabs.DistSlab(g, rank, world, "weno5", overlap=True), "nccl-overlap"
            for q in range(W):
                runner.step(stepper, dt, q)
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # the overlapped NCCL path (interior rows, then the strips) is timed as
    # the runner runs it, one event pair per step; otherwise one per stage
    # launch (the fused peer push and single-GPU runs are whole-stage launches)
    per_step = halo == "nccl-overlap"
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(K if per_step else ns * K)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    t_start.record(stream)
    i = 0
    for q in range(K):
        if per_step:
            evs[i][0].record(stream)
            runner.step(stepper, dt, W + q)
            evs[i][1].record(stream)
            i += 1
            continue
        for st in range(ns):
            runner.exchange(g.stage_input(stepper, st))
            evs[i][0].record(stream)
            g.launch_stage(stepper, st, dt, W + q)
            evs[i][1].record(stream)
            i += 1
    t_end.record(stream)
    torch.cuda.synchronize()
    total_ms = t_start.elapsed_time(t_end)
    if world > 1:
        t = torch.tensor([total_ms], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    stage_ms = np.array([a.elapsed_time(b) for a, b in evs]).reshape(K, 1 if per_step else ns)
    blown, _ = g.status()
    if blown:
        raise RuntimeError(f"benchmark state blew up ({mode})")
    value = world * P * ns * K / (total_ms / 1000.0)
    # algorithmic bytes per step: RK3 stage 1 136 B/pt, stages
    # 2-3 168 B/pt (fp64 state 32 B + coefficients 72 B); RK(10,4) 1520 B/pt;
    # double-double tiers twice that
    bytes_per_step = P * (472 if ns == 3 else 1520) * (2 if mode.startswith("dd") else 1)
    kern_ms = float(stage_ms.sum())
    achieved = bytes_per_step * K / (kern_ms / 1000.0) / 1e9
    return g, dict(value=value, total_ms=total_ms, stage_ms=stage_ms, achieved_gbs=achieved,
                   kern_ms=kern_ms, P=P, dt=dt, K=K, halo=halo, runner=runner)


def sustained_mode(g, args, prob, dt, torch, clocks_cls, dev, warm_s=1.0, timed_s=2.5,
                   tau_chunk=20.0):
    """The headline tier under sustained load: whole SSP-RK3 steps replayed
    back to back (hwg_launch_steps, CUDA graphs) for >= warm_s untimed, then
    >= timed_s timed with CUDA events and its own clock record (the 20-step
    burst sits inside the power-cap transient).  The extremal
    Kerr m=2 pulse grows by ~e per 3 units of tau on the fast tiers as in the
    reference (tools/probe_growth.py), so a small grid, which needs ~10^5 steps
    to fill the window, restarts from the initial state every tau_chunk
    (a host set_state between timed chunks, outside the events; the C5 grid
    never needs one)."""
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)  # e2e_mode may have moved the handle to its own stream
    P = prob["nrho"] * prob["ntheta"]
    from paper_2010_04760_b200 import synthetic
    u0 = synthetic.initial_state(prob)
    g.set_state(u0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.launch_steps("ssprk33", dt, 0, 20)
    e0.record(stream)
    g.launch_steps("ssprk33", dt, 20, 20)
    e1.record(stream)
    torch.cuda.synchronize()
    per = max(e0.elapsed_time(e1) / 20.0, 1e-3)
    nw = min(100000, max(20, int(warm_s * 1e3 / per)))
    nt = min(100000, max(20, int(timed_s * 1e3 / per)))
    chunk = max(20, int(tau_chunk / dt))
    state = {"step": 40, "restarts": 0}

    def run(n, timed):
        """n steps in chunks that stay within tau_chunk of a (re)start."""
        ms = 0.0
        while n > 0:
            k = min(n, chunk)
            if state["step"] + k > chunk:  # restart the pulse (untimed)
                torch.cuda.synchronize()
                g.set_state(u0)
                state["step"] = 0
                state["restarts"] += 1
            if timed:
                e0.record(stream)
            g.launch_steps("ssprk33", dt, state["step"], k)
            if timed:
                e1.record(stream)
                torch.cuda.synchronize()
                ms += e0.elapsed_time(e1)
                if g.status()[0]:
                    raise RuntimeError("sustained run blew up")
            state["step"] += k
            n -= k
        return ms

    ck = clocks_cls(dev)
    ck.start()
    run(nw, False)
    ck.mark()
    ms = run(nt, True)
    ck.mark()
    ck.stop()
    restarts = state["restarts"]
    return {"value": P * 3 * nt / (ms / 1e3), "ms_per_step": ms / nt, "steps": nt,
            "warm_steps": nw, "timed_s": ms / 1e3, "restarts": restarts,
            "clocks": ck.summary()}


def _e2e_job(g, u, out, dt, q, runner=None):
    """One end-to-end step through the C ABI with host buffers: hwg_set_state
    (host FieldLayout -> device), one SSP-RK3 step, hwg_get_state (device ->
    host FieldLayout, ghosts filled).  Returns the three phase times."""
    from paper_2010_04760_b200.hwgpu import _lib, _p
    a = time.perf_counter()
    g.set_state(u)
    if runner is not None and hasattr(runner, "prime"):
        runner.prime()  # fused-halo slabs: halos of the uploaded state
    b = time.perf_counter()
    if runner is None:
        g.launch_steps("ssprk33", dt, q, 1)
    else:
        runner.step("ssprk33", dt, q)
    g.synchronize()
    c = time.perf_counter()
    g._chk(_lib.hwg_get_state(g.h, _p(out)))
    return b - a, c - b, time.perf_counter() - c


def e2e_mode(g, args, prob, world, rank, torch, dist, dt, runner=None):
    """Same metric through the C ABI with HOST buffers (pinned, as the
    contract allows): every step uploads its host state, advances one RK3 step
    and reads the whole state back (_e2e_job).  The steps are independent
    jobs (same input), so on one GPU two handles on their own streams run them
    two-deep from two host threads: job q+1's upload (H2D) overlaps job q's
    read-back (D2H), both PCIe directions busy.  Multi-GPU slabs run them
    serially (the halo exchange is one NCCL sequence per process)."""
    import threading
    from paper_2010_04760_b200 import hwgpu, slabs, synthetic
    u0 = synthetic.initial_state(prob)
    ke = max(1, min(args.e2e_steps, args.steps))
    lanes = max(1, min(args.e2e_lanes, ke)) if world == 1 else 1
    hs = [g]
    for _ in range(lanes - 1):
        h = hwgpu.GpuEvolution(prob["nrho"], prob["ntheta"], prob["drho"], prob["dtheta"],
                               prob["parity"], prob["coef"], prob["cotth"], g.spec,
                               device=torch.cuda.current_device(), coef_ld=prob["nrho"],
                               coef_row0=0)
        hs.append(h)
    bufs = []
    for h in hs:
        if lanes > 1:
            h.set_stream(None)  # each lane on its own stream
        u = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
        u[...] = u0
        out = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
        bufs.append((u, out))
        _e2e_job(h, u, out, dt, 0)  # warm the staging buffers and graphs
    runner = runner if world > 1 else None
    if world > 1:
        dist.barrier()
    times = [[0.0, 0.0, 0.0] for _ in hs]

    def lane(i):
        for q in range(i, ke, lanes):
            r = _e2e_job(hs[i], bufs[i][0], bufs[i][1], dt, q, runner)
            for k in range(3):
                times[i][k] += r[k]

    t0 = time.perf_counter()
    if lanes == 1:
        lane(0)
    else:
        th = [threading.Thread(target=lane, args=(i,)) for i in range(lanes)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    wall = time.perf_counter() - t0
    for h in hs[1:]:
        h.close()
    if lanes > 1:
        g.set_stream(torch.cuda.current_stream().cuda_stream)
    if world > 1:
        t = torch.tensor([wall], device=f"cuda:{torch.cuda.current_device()}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        wall = float(t.item())
    P = prob["nrho"] * prob["ntheta"]
    tot = [sum(t[k] for t in times) / ke for k in range(3)]
    u = bufs[0][0]
    return dict(value=world * P * 3 * ke / wall, steps=ke, h2d=int(u.nbytes), d2h=int(u.nbytes),
                lanes=lanes, ms=dict(set_state=1e3 * tot[0], step=1e3 * tot[1],
                                     get_state=1e3 * tot[2], wall_per_step=1e3 * wall / ke))


def e2e_advance_mode(g, args, prob, dt, torch, K=None, every=1):
    """The drop-in's own usage of the boundary (the reference's driver calls
    advance_steps once per run, driver.cpp:93): one hwg_advance call over K
    steps with the HOST state in and out (pinned FieldLayout, hwg_set_state /
    hwg_get_state inside the timed region) and the observers read back to the
    host through the hook every `every` steps (the reference's driver
    samples every round(0.25/dt) steps, driver.cpp:40-49).  Reported beside
    the strict per-step round trip (e2e)."""
    from paper_2010_04760_b200 import synthetic
    from paper_2010_04760_b200.hwgpu import HwgObservables, _lib, _p
    nrho, nth = prob["nrho"], prob["ntheta"]
    hw = np.zeros((4, 8))
    hw[0, 0] = 1.0                                   # Phi(rho_min)
    hw[1, :4] = np.array([-11.0, 18.0, -9.0, 2.0]) / (6.0 * prob["drho"])  # one-sided d/drho
    g.set_observers(nth // 2, 0, hw, nrho // 2, np.full(nth, 1.0 / nth))
    u = torch.empty(g.shape, dtype=torch.float64, pin_memory=True).numpy()
    u[...] = synthetic.initial_state(prob)
    out = torch.empty(g.shape, dtype=torch.float64, pin_memory=True).numpy()
    K = args.steps if K is None else K
    seen = []
    hook = lambda step, tau, obs: seen.append(obs["dphi"][0])  # noqa: E731
    g.set_state(u)
    g.advance("ssprk33", dt, 0, 2, every=every, hook=hook)      # warm
    g._chk(_lib.hwg_get_state(g.h, _p(out)))
    seen.clear()
    t0 = time.perf_counter()
    g.set_state(u)
    st = g.advance("ssprk33", dt, 0, K, every=every, hook=hook)
    g._chk(_lib.hwg_get_state(g.h, _p(out)))
    wall = time.perf_counter() - t0
    nhook = len(range(0, K, every)) + 1  # s % every == 0 for s < K, and s == K
    if st["blew_up"] or st["steps_done"] != K or len(seen) != nhook:
        raise RuntimeError(f"e2e advance: {st}, {len(seen)} hook calls (expected {nhook})")
    ob = ctypes.sizeof(HwgObservables)
    return {"value": nrho * nth * 3 * K / wall, "unit": UNIT,
            "h2d_bytes_per_step": u.nbytes / K,
            "d2h_bytes_per_step": (out.nbytes + len(seen) * ob) / K, "steps": K,
            "hook_every": every, "hook_calls": len(seen),
            "path": f"C ABI hwg_set_state + hwg_advance(K steps, observers to the host every "
                    f"{every} step(s)) + hwg_get_state, pinned host FieldLayout fp64"}


# the other BASELINE shapes (parity-test configurations; not the headline):
# (label, nrho, ntheta, scheme, mode)
CONFIG_SHAPES = [
    ("C1 1024x64 weno5 f64", 1024, 64, "weno5", "f64"),
    ("C2 4096x128 weno5 mixed", 4096, 128, "weno5", "mixed"),
    ("C3 16384x128 weno5 mixed", 16384, 128, "weno5", "mixed"),
    ("C3 16384x128 weno5 f64", 16384, 128, "weno5", "f64"),
    ("C4 4096x128 fd6ko", 4096, 128, "fd6ko", "mixed"),
]
# their physics: the reference's planes assembled on the GPU
CONFIG_PHYSICS = {
    "C1": dict(a=0.0, spin=0, mmode=0),
    "C2": dict(a=1.0, spin=-2, mmode=2),
    "C3": dict(a=0.9, spin=-2, mmode=0),
    "C4": dict(a=1.0, spin=-2, mmode=2),
}


def config_rates(torch):
    """Stage-updates/s of the same kernels at the other BASELINE shapes, one
    handle each, whole SSP-RK3 steps replayed as a CUDA graph
    (hwg_launch_steps) for ~50 ms after 5 warm-up steps.  C1-C4 fit in the
    126 MB L2 (no flush: the point is the resident-grid rate) and are
    launch/latency bound rather than HBM bound."""
    from paper_2010_04760_b200 import hwgpu, planes, synthetic
    out = {}
    stream = torch.cuda.current_stream()
    for label, n, nt, sch, mode in CONFIG_SHAPES:
        prob = planes.problem_or_synthetic(n, nt, **CONFIG_PHYSICS[label[:2]])
        g = hwgpu.GpuEvolution(n, nt, prob["drho"], prob["dtheta"], prob["parity"],
                               prob["coef"], prob["cotth"], hwgpu.SchemeSpec(sch, mode))
        g.set_stream(stream.cuda_stream)
        g.set_state(synthetic.initial_state(prob))
        dt = synthetic.select_dt(prob)
        g.launch_steps("ssprk33", dt, 0, 5)
        torch.cuda.synchronize()
        K = int(min(5000, max(20, 0.05 * 2.5e10 / (3 * n * nt))))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        g.launch_steps("ssprk33", dt, 5, K)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        blown, _ = g.status()
        g.close()
        if blown:
            raise RuntimeError(f"{label}: state blew up")
        out[label] = {"value": n * nt * 3 * K / (ms / 1e3), "ms_per_step": ms / K, "steps": K,
                      "l2": "resident (grid < L2)" if n * nt * 168 < 100e6 else "streams"}
    return out


def fp64_peak():
    """Measured FP64 lane-operations/s of this B200 (tools/fp_peaks.cu, the
    DFMA/DADD throughput kernels; profiles/r02_fp_peaks.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_fp_peaks.json")) as f:
            p = json.load(f)
        return min(p["dfma"]["lane_ops_per_s"], p["dadd"]["lane_ops_per_s"]), "measured"
    except Exception:
        return 1.8e13, "fallback"


def mode_record(m, r, peak):
    """Per-tier line entry.  The fp64 / mixed tiers are HBM-bound: frac of
    the copy peak.  The double-double tiers are FP64-pipe bound: their
    roofline is the FP64 pipe — FP64 lane operations per point-stage (ncu
    count of the SSP-RK3 middle-stage kernel, profiles/dd_fp64_ops.json)
    x updates/s over the measured FP64 peak — and the HBM fraction is kept
    for reference only."""
    rec = {"value": r["value"], "ms_per_step": r["total_ms"] / r["K"], "steps": r["K"],
           "stepper": "ssprk104" if m.endswith("ssprk104") else "ssprk33",
           "stage_kernel_gbs": r["achieved_gbs"], "frac": r["achieved_gbs"] / peak,
           "step_or_stage_ms_mean": [float(x) for x in r["stage_ms"].mean(axis=0)],
           "halo": r["halo"]}
    if m.startswith("dd"):
        try:
            with open(os.path.join(ROOT, "profiles", "dd_fp64_ops.json")) as f:
                ops = json.load(f)[m]["fp64_lane_ops_per_point_stage"]
        except Exception:
            ops = None
        fpk, src = fp64_peak()
        rec["roofline"] = {"bound": "fp64", "unit": "FP64 lane-ops/s", "peak": fpk,
                           "peak_source": src, "ops_per_point_stage": ops,
                           "achieved": ops * r["value"] if ops else None,
                           "frac": ops * r["value"] / fpk if ops else None}
        # the measured ceiling of DD code at the kernel's occupancy (8 warps
        # per SM): the WENO5 DD interface alone, register-resident, one chain
        # per thread (tools/dd_peak.cu, profiles/r02_dd_peak.json)
        try:
            with open(os.path.join(ROOT, "profiles", "r02_dd_peak.json")) as f:
                runs = json.load(f)["runs"]
            name = "weno5_dd mixed" if m == "dd-mixed" else "weno5_dd full"
            ceil = next(x["frac_of_dfma_peak"] for x in runs if x["kernel"] == name
                        and x["warps_per_sm"] == 8 and x["chains_per_thread"] == 1)
            rec["roofline"]["dd_interface_ceiling"] = ceil
            if ops:
                rec["roofline"]["frac_of_dd_ceiling"] = rec["roofline"]["frac"] / ceil
        except Exception:
            pass
        rec["frac_hbm_for_reference"] = rec.pop("frac")
    return rec


def run_b200(args):
    import torch
    import torch.distributed as dist
    world, rank, local = dist_env()
    if world > 1:
        # test plumbing only (tests/test_gpu_bench.py): all ranks on GPU 0 with
        # a host-only backend, so the multi-rank control flow (slab
        # partition, halo exchange, max-over-ranks timing, rank-0 line) runs
        # on a 1-GPU box; never the fused push there (kernels would wait on
        # each other on one GPU) — --halo nccl with DistSlab's staged exchange
        backend = os.environ.get("HWG_BENCH_BACKEND", "nccl")
        local_dev = 0 if os.environ.get("HWG_BENCH_ONE_GPU") else local
        torch.cuda.set_device(local_dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_dev}"))
        else:
            if args.halo == "peer":
                raise SystemExit("HWG_BENCH_BACKEND=gloo needs --halo nccl")
            dist.init_process_group(backend)
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_2010_04760_b200 import planes, slabs

    ng = args.nrho * world
    off, cnt = slabs.partition(ng, world)[rank]
    t0 = time.perf_counter()
    prob = planes.problem_or_synthetic(cnt, args.ntheta, rho_offset=off, nrho_global=ng, device=dev)
    setup_s = time.perf_counter() - t0
    log(f"coefficient planes assembled on the GPU in {setup_s:.2f} s")
    if world > 1:  # one dt for all slabs: the whole grid's max speed
        ms = torch.tensor([prob["max_speed"]], dtype=torch.float64,
                          device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        prob["max_speed"] = float(ms.item())
    clocks = ClockSampler(dev)
    clocks.start()
    results = {}
    # headline mode last so its clock window is the one reported
    modes = ["f64", "mixed"] if args.mode == "mixed" else ["mixed", "f64"]
    handles = {}
    for mode in modes:
        if mode == modes[-1]:
            clocks.mark()
        log(f"time_mode {mode}")
        g, r = time_mode(args, mode, prob, world, rank, dev, torch, dist)
        if mode == modes[-1]:
            clocks.mark()
        results[mode] = r
        handles[mode] = g
    clocks.stop()
    head = results[args.mode]
    g = handles[args.mode]
    for m in list(handles):
        if m != args.mode:
            handles.pop(m).close()
    # the reference's production stepper (all proj/configs/*.ini use ssprk104)
    log("time_mode ssprk104")
    g4, r = time_mode(args, args.mode, prob, world, rank, dev, torch, dist,
                      steps=max(1, args.steps // 3), stepper="ssprk104")
    g4.close()
    results[f"{args.mode}-ssprk104"] = r
    # the reference's own precisions (double-double tiers, bitwise equal to the
    # reference library): the paper's mixed-vs-full experiment on B200
    if not args.no_dd:
        for mode in ("dd-mixed", "dd-full"):
            log(f"time_mode {mode}")
            gd, r = time_mode(args, mode, prob, world, rank, dev, torch, dist,
                              steps=max(1, min(3, args.steps)), warmup=1)
            gd.close()
            results[mode] = r
    log("e2e")
    e2e = e2e_mode(g, args, prob, world, rank, torch, dist, head["dt"], head["runner"])
    log("e2e_advance")
    e2e_adv = e2e_advance_mode(g, args, prob, head["dt"], torch) if world == 1 else None
    # the drop-in at the reference driver's observer cadence, round(0.25/dt)
    # steps (driver.cpp:40-49), over two sampling periods
    e2e_prod = None
    if world == 1 and not args.no_sustained:
        dt_hi = head["dt"][0] if isinstance(head["dt"], tuple) else float(head["dt"])
        every = max(1, int(round(0.25 / dt_hi)))
        log(f"e2e_advance production cadence every {every}")
        e2e_prod = e2e_advance_mode(g, args, prob, head["dt"], torch, K=2 * every, every=every)
    sustained = None
    if world == 1 and not args.no_sustained:
        log("sustained")
        sustained = sustained_mode(g, args, prob, head["dt"], torch, ClockSampler, dev)
    log("other configs")
    shapes = config_rates(torch) if world == 1 and not args.no_configs else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        log("cpu baseline")
        cpu = cpu_reference_rate(args.nrho, args.ntheta)
        log("done")
    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return 0
    peak, src = peaks()
    traffic = None
    tf = os.path.join(ROOT, "profiles", "stage_kernel_traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            key = f"{args.mode}_{args.nrho}x{args.ntheta}"
            traffic = tj.get(key)
        except Exception:
            traffic = None
    pipes = None
    pf = os.path.join(ROOT, "profiles", "stage_kernel_pipes.json")
    if os.path.exists(pf):
        try:
            pipes = json.load(open(pf)).get(f"{args.mode}_{args.nrho}x{args.ntheta}")
        except Exception:
            pipes = None
    ach = head["achieved_gbs"]
    info = g.launch_info()
    K = args.steps
    line = {
        "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": head["total_ms"] / K, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 state, fp32 WENO weights" if args.mode == "mixed" else "f64",
        "data": ("the reference's extremal-Kerr (a=M, s=-2, m=2) coefficient planes on the "
                 f"BASELINE C5 grid, assembled on the GPU in {setup_s:.2f} s by the reference's "
                 "generated wave_op_coeffs kernels in double-double (hwg_assemble_coefficients, "
                 "fp64 grid); synthetic initial state (Gaussian pulse)")
                if prob["planes"] == "device-assembled" else
                ("synthetic coefficient planes with the reference's sign structure (this "
                 "libhwgpu.so was built without the reference headers); synthetic initial state"),
        "config": {"workload": f"C5 shape {args.nrho}x{args.ntheta} per GPU (radial slabs of "
                               f"{args.nrho * world}x{args.ntheta}), WENO5 {args.mode}, SSP-RK3",
                   "grid_points_per_gpu": head["P"], "stages_per_step": 3,
                   "l2": "inputs larger than L2 (no flush needed)",
                   "parallelism": f"rho-slabs x{world}",
                   "halo": head["halo"]},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak, "traffic": traffic, "peak_source": src,
                     "kernel": "hwg::stage_kernel<WENO5>",
                     "bytes_per_point_stage": 157.33,
                     # FP64 / FP32 / XU pipe and issue utilisation of the
                     # three SSP-RK3 stage kernels (ncu --set full; the
                     # weight computation's pipes, north_star)
                     "pipes": pipes,
                     # secondary denominator: the B200 HBM3e datasheet figure
                     "frac_of_spec_8000_gbs": ach / 8000.0},
        "clocks": clocks.summary(),
        "e2e": {"value": e2e["value"], "unit": UNIT, "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "steps": e2e["steps"], "lanes": e2e["lanes"],
                "ms_per_step": e2e["ms"],
                "path": "C ABI hwg_set_state + 1 RK3 step + hwg_get_state (pinned host "
                        "FieldLayout fp64); independent jobs, 'lanes' in flight"},
        "e2e_advance": e2e_adv,
        "e2e_advance_production": e2e_prod,
        "sustained": None if sustained is None else {
            **sustained, "roofline_frac": sustained["value"] * 157.33 / 1e9 / peak,
            "vs_burst": sustained["value"] / head["value"]},
        "other_configs": shapes,
        "gpu_launches": 3 * K,
        "launch": info,
        "modes": {m: mode_record(m, r, peak) for m, r in results.items()},
        "mixed_vs_fp64_speedup": results["mixed"]["value"] / results["f64"]["value"],
    }
    if "dd-full" in results:
        line["dd_mixed_vs_dd_full_speedup"] = (results["dd-mixed"]["value"] /
                                               results["dd-full"]["value"])
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="mixed", choices=["mixed", "f64"])
    ap.add_argument("--nrho", type=int, default=65536)
    ap.add_argument("--ntheta", type=int, default=512)
    ap.add_argument("--e2e-steps", type=int, default=32,
                    help="independent e2e jobs timed (more jobs amortise the PCIe pipeline fill and drain)")
    ap.add_argument("--e2e-lanes", type=int, default=4,
                    help="independent e2e jobs in flight on one GPU (own handle + stream each)")
    ap.add_argument("--halo", default="peer", choices=["peer", "nccl"],
                    help="N > 1 slab halos: fused push over NVLink peer memory, or NCCL P2P")
    ap.add_argument("--ref-steps", type=int, default=3,
                    help="--impl reference: timed reference steps cap (seconds each at 65536x512)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-dd", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    ap.add_argument("--no-sustained", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
