"""Benchmark: Method-S3 stochastic-MFB sweep on B200.

A "step" is one full S3 sweep of the workload config (default: BASELINE
configs[1] = configs/cfg2.json): KL fields for every local realization,
assembly + factor + multi-RHS solve of every (subdomain, local realization)
system, the batched interface CG over all collocation points, and the
moments. `value` = collocation realizations/s with the problem resident in
HBM (device time, CUDA events); `e2e` = the same metric through the public
API `run_method(problem, grid, "S3", tol)` with host inputs and host
results (H2D of the step's KL/collocation tables, D2H of lambdas, residual
histories and moments inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2]
    python bench.py --impl reference ...   # the reference CPU algorithm (oracle port)

Under torchrun (N > 1) every rank runs the same sweep on its own GPU
(weak scaling, replicas); timing is the max over ranks.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--tol", type=float, default=1e-11)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-s2", action="store_true",
                    help="skip the deterministic-MFB (S2) comparison sweep")
    return ap.parse_args()


def _config_path(name):
    return name if name.endswith(".json") else os.path.join(ROOT, "configs", name + ".json")


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True,
                    timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001 - clocks are best effort
                pass
            self._stop.wait(0.1)

    def prime(self):
        """One query before any timing: the first nvidia-smi call on a box
        (driver/NVML initialisation) disturbs GPU work running beside it
        (measured: 12 ms instead of 6 ms per cfg2 sweep), later ones do not."""
        try:
            subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                            "--format=csv,noheader,nounits"], capture_output=True, timeout=30)
        except Exception:  # noqa: BLE001 - clocks are best effort
            pass

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.samples)}


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    peaks = {}
    if os.path.exists(path):
        with open(path) as fh:
            peaks = json.load(fh)
    fp64 = None
    fpath = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(fpath):
        with open(fpath) as fh:
            fp64 = json.load(fh)
    return peaks, fp64


def _traffic(kind, config):
    """DRAM bytes per launch of a kernel kind from the committed ncu capture
    (only for the workload that capture was taken on)."""
    path = os.path.join(ROOT, "profiles", "r01", "traffic.json")
    if not os.path.exists(path):
        return None, None
    with open(path) as fh:
        t = json.load(fh).get(kind)
    if not t or t.get("config") != config:
        return None, None
    return t["dram_bytes_per_launch"], t["source"]


def s2_comparison(plan, problem, grid, tol, max_iter, flush, steps=2):
    """BASELINE configs[1]: "compare deterministic MFB and stochastic MFB on
    identical inputs" -- the same workload swept with Method S2 (a flux basis
    per subdomain per realization, Stokes included) on the device, device
    time per sweep (CUDA events, L2 flushed) and end to end via run_method."""
    import torch
    from paper_1802_06263_b200.interface import SweepEngine, run_method

    def sweep():
        e = SweepEngine(plan, method="S2")
        e.kl_fields()
        e.build_bases()
        lam, iters, status, hist, _ = e.solve_points(tol, max_iter)
        e.moments(lam)
        return iters

    sweep()
    ms = []
    for _ in range(steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        iters = sweep()
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    run_method(problem, grid, method="S2", tol=tol)
    t = time.perf_counter()
    for _ in range(steps):
        run_method(problem, grid, method="S2", tol=tol)
    e2e = (time.perf_counter() - t) / steps
    systems = plan.n_sub * grid.n_real
    return {"method": "S2 (deterministic MFB)", "value": grid.n_real / (np.mean(ms) / 1e3),
            "unit": "realizations/s", "ms_per_step": float(np.mean(ms)), "steps": steps,
            "systems_per_sweep": systems, "cg_iters_mean": float(iters.float().mean().item()),
            "e2e": {"value": grid.n_real / e2e, "unit": "realizations/s",
                    "api": "run_method(problem, grid, 'S2', tol)"}}


def s1_comparison(plan, problem, grid, tol, hbm_peak, steps=1):
    """the same workload swept with Method S1 (matrix-free:
    per-realization factors, one batched star solve per CG iteration) end to
    end through run_method. The star solves stream the stored factors from
    HBM every iteration: algorithmic bytes = sum over points of N_iter(k) x
    (multiplier panels + U band of every subdomain), over the CG phase."""
    from paper_1802_06263_b200.interface import run_method
    run_method(problem, grid, method="S1", tol=tol)
    t = time.perf_counter()
    for _ in range(steps):
        res = run_method(problem, grid, method="S1", tol=tol)
    e2e = (time.perf_counter() - t) / steps
    it = np.array(res.stats.cg_iters, dtype=np.int64)
    per_pt = sum(8 * ((p.n + 15) // 16) * (p.kl + 16) * 16 + 8 * p.n * (p.kl + p.ku)
                 for p in plan.patterns)
    cg_s = res.timings["cg"]
    ach = float(it.sum()) * per_pt / cg_s / 1e9
    return {"method": "S1 (matrix-free)", "value": grid.n_real / e2e, "unit": "realizations/s",
            "api": "run_method(problem, grid, 'S1', tol)", "steps": steps,
            "cg_iters_mean": float(it.mean()), "cg_iters_max": int(it.max()),
            "phases_s": {"bases": res.timings["bases"], "cg": cg_s,
                         "recovery_moments": res.timings["moments"]},
            "star_solve_roofline": {"bound": "hbm", "achieved": ach, "peak": hbm_peak,
                                    "unit": "GB/s", "frac": ach / hbm_peak if hbm_peak else None,
                                    "bytes_per_point_iteration": per_pt}}


def cpu_baseline(cfg_path, tol, sample_points=None):
    """Reference CPU algorithm (oracle port of sdmortar S3), 1 thread."""
    from threadpoolctl import threadpool_limits

    from oracle import s3_cpu
    from paper_1802_06263_b200.adapter import load_config
    problem, grid, _ = load_config(cfg_path)
    pts = None if sample_points is None else list(range(min(sample_points, grid.n_real)))
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        ops, bases = s3_cpu.prepare_s3(problem, grid)
        t_pre = time.perf_counter() - t0
        solves = sum(len(b) * b[0][1].shape[0] for b in bases.values())
        t1 = time.perf_counter()
        _run_points(s3_cpu, problem, grid, ops, bases, tol, pts)
        t_main = time.perf_counter() - t1
    n_done = grid.n_real if pts is None else len(pts)
    per_point = t_main / max(n_done, 1)
    est_total = t_pre + per_point * grid.n_real
    return {
        "realizations_per_s": grid.n_real / est_total,
        "basis_local_solves_per_s": solves / t_pre,
        "pre_loop_s": t_pre, "main_loop_s": t_main, "points_timed": n_done,
        "n_real": grid.n_real, "extrapolated": pts is not None,
    }


def _run_points(s3_cpu, problem, grid, ops, bases, tol, pts):
    """The S3 main loop of the oracle for a subset of points (no re-prepare)."""
    n_sub = problem.layout.n_subdomains
    space = problem.space
    acc = s3_cpu.Moments()
    for k in (range(grid.n_real) if pts is None else pts):
        loc = [s3_cpu.local_of(problem, grid, s, k) for s in range(n_sub)]
        pick_ops = [ops[s][loc[s]] for s in range(n_sub)]
        pick_b = [bases[s][loc[s]] for s in range(n_sub)]

        def apply_fn(lam, pick_b=pick_b):
            out = np.zeros(space.n_dof)
            for dofs, B in pick_b:
                out[dofs] += B @ lam[dofs]
            return out

        bars, entries = [], []
        for s in range(n_sub):
            u, p = s3_cpu.bar_solve(pick_ops[s])
            bars.append((u, p))
            entries += s3_cpu.side_values(problem, s, pick_ops[s], u)
        g = s3_cpu.jump(space, entries)
        lam, _, _ = s3_cpu.cg_solve(apply_fn, g, tol=tol)
        fields = {"lambda": lam}
        for s in range(n_sub):
            us, ps = s3_cpu.star_solve(problem, s, pick_ops[s], lam)
            f = pick_ops[s].postprocess(bars[s][0] + us, bars[s][1] + ps)
            for name, arr in f.items():
                fields[f"{s}:{name}"] = arr
        acc.add(grid.weights[k], fields)
    return acc


def run_reference(a):
    ws, rank, _ = _dist()
    if rank != 0:
        return
    from paper_1802_06263_b200.adapter import load_config
    cfg_path = _config_path(a.config)
    problem, grid, _ = load_config(cfg_path)
    cores = len(os.sched_getaffinity(0))
    # each step: full pre-loop + a bounded prefix of the main loop, extrapolated
    sample = 8
    vals = []
    t_all = time.perf_counter()
    for i in range(a.warmup + a.steps):
        from oracle import s3_cpu
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=cores):
            t0 = time.perf_counter()
            ops, bases = s3_cpu.prepare_s3(problem, grid, workers=cores)
            t_pre = time.perf_counter() - t0
            t1 = time.perf_counter()
            _run_points(s3_cpu, problem, grid, ops, bases, a.tol, list(range(min(sample, grid.n_real))))
            t_main = time.perf_counter() - t1
        n_done = min(sample, grid.n_real)
        est = t_pre + t_main / n_done * grid.n_real
        if i >= a.warmup:
            vals.append(grid.n_real / est)
    v = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": f"collocation realizations/s (S3 sweep, {a.config})",
        "value": v, "unit": "realizations/s", "n_gpus": ws, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1000.0 * grid.n_real / v,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (deterministic collocation grid of the config)",
        "config": {"workload": a.config, "n_real": grid.n_real, "tol": a.tol},
        "cpu_baseline": {"value": v, "unit": "realizations/s", "cores": cores,
                         "kind": "port",
                         "sample": f"oracle/s3_cpu.py (restated sdmortar S3: SuperLU + numpy CG), "
                                   f"full pre-loop on a {cores}-thread pool (the reference's "
                                   f"workers) + first {sample} of {grid.n_real} points per "
                                   f"step, extrapolated to the full sweep"},
        "e2e": {"value": v, "unit": "realizations/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
    }
    print(json.dumps(line), flush=True)


def run_ours(a):
    import torch
    ws, rank, local = _dist()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    from paper_1802_06263_b200 import _build
    from paper_1802_06263_b200.adapter import load_config
    from paper_1802_06263_b200.interface import SweepEngine, get_plan, run_method
    _build.build()
    cfg_path = _config_path(a.config)
    problem, grid, _ = load_config(cfg_path)
    nl = problem.space.n_dof
    max_iter = max(50, 10 * nl)
    t0 = time.perf_counter()
    plan = get_plan(problem, grid)
    plan_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")   # > 126 MB L2

    if ws > 1:
        import torch.distributed as dist

        from paper_1802_06263_b200.distributed import (DeviceShardEngine, run_method_distributed,
                                                       run_sharded)

        def step(eng):
            out = run_sharded(eng, grid.n_real, nl, a.tol, max_iter, dist, rank, ws)
            return out

        def new_engine():
            e = DeviceShardEngine(plan)
            e.eng.timing = True
            return e
    else:
        def step(eng):
            eng.kl_fields()
            eng.build_bases()
            lam, iters, status, hist, _ = eng.solve_points(a.tol, max_iter)
            mom = eng.moments(lam)
            return lam, iters, status, mom

        def new_engine():
            e = SweepEngine(plan)
            e.timing = True
            return e

    def timed_step():
        e = new_engine()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        step(e)
        t1.record(stream)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1)

    clocks = ClockSampler(local)
    clocks.prime()
    warm = [timed_step() for _ in range(a.warmup)]
    # Keep warming up -- beyond the W requested, reported as
    # warmup_extra_steps -- until the last three warm-up steps agree within
    # 3% and at least 0.3 s has passed (at most 20 s): the timed steps then
    # start from a steady state whatever state the process found the GPU in.
    extra, t_w = 0, time.perf_counter()
    while True:
        last = warm[-3:]
        done = (len(last) == 3 and max(last) <= 1.03 * min(last)
                and time.perf_counter() - t_w >= 0.3) or time.perf_counter() - t_w > 20.0
        if ws > 1:                  # the ranks stop together (collectives inside a step)
            flag = torch.tensor([1 if done else 0], device="cuda")
            torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
            done = bool(flag.item())
        if done:
            break
        warm.append(timed_step())
        extra += 1
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    dev_ms, e2e_s = [], []
    solve_ms, cg_ms, bases_ms, launches = [], [], [], 0
    cg_name = "cg"
    iters_host = None
    with clocks:
        for _ in range(a.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if ws > 1:
                torch.distributed.barrier()
            eng = new_engine()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            out = step(eng)                       # moments include D2H of the results
            e1.record(stream)
            torch.cuda.synchronize()
            dev_ms.append(e0.elapsed_time(e1))
            core = eng.eng if ws > 1 else eng
            launches = core.launches
            for kind, s0, s1, fl, sfl in core.solve_events:
                solve_ms.append((kind, s0.elapsed_time(s1), fl, sfl))
            cg_name = getattr(core, "cg_kernel_name", "cg")
            for b0, b1 in core.bases_events:
                bases_ms.append(b0.elapsed_time(b1))
            for c0, c1, _ in core.cg_events:
                cg_ms.append(c0.elapsed_time(c1))
            if ws > 1:
                iters_host = out[2] if out is not None else np.zeros(1)
            else:
                iters_host = out[1].cpu().numpy()
            core.check_info()
        # end-to-end through the public API, host in / host out (one untimed
        # call first: first-use costs of the host-side packing stay outside)
        if ws > 1:
            run_method_distributed(problem, grid, tol=a.tol)
        else:
            run_method(problem, grid, method="S3", tol=a.tol)
        torch.cuda.synchronize()
        for _ in range(a.steps):
            flush.fill_(1)
            torch.cuda.synchronize()
            if ws > 1:
                torch.distributed.barrier()
            t = time.perf_counter()
            if ws > 1:
                res = run_method_distributed(problem, grid, tol=a.tol)
                torch.cuda.synchronize()
            else:
                res = run_method(problem, grid, method="S3", tol=a.tol)
            e2e_s.append(time.perf_counter() - t)
    if ws > 1:
        tmax = torch.tensor([sum(dev_ms), sum(e2e_s)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tmax, op=torch.distributed.ReduceOp.MAX)
        tot_ms, tot_e2e = float(tmax[0]), float(tmax[1])
    else:
        tot_ms, tot_e2e = sum(dev_ms), sum(e2e_s)
    ms_step = tot_ms / a.steps
    # ws > 1: the ranks share ONE sweep (points and subdomains sharded)
    value = grid.n_real / (ms_step / 1000.0)
    e2e_val = grid.n_real / (tot_e2e / a.steps)
    systems = plan.s3_systems()
    local_solves = int(sum(int(plan.ndof[s]) for s, _ in systems))
    peaks, fp64 = _peaks()
    # dominant basis kernel of the step (per-kind CUDA-event totals over the timed steps)
    kinds = {}
    for kind, ms, fl, sfl in solve_ms:
        k = kinds.setdefault(kind, [0.0, 0.0, 0.0, 0])
        k[0] += ms
        k[1] += fl
        k[2] += sfl
        k[3] += 1
    dom = max(kinds, key=lambda x: kinds[x][0]) if kinds else None
    peak = fp64["dmma_tflops"] if fp64 else None
    roof = None
    if dom:
        t_ms, fl, sfl, cnt = kinds[dom]
        # achieved = SURVEY 8(d) algorithmic flops (F = 2 n w^2 + 4 n w N_dof of the banded
        # mixed system) / kernel time; the flops the kernel actually executes are reported
        # beside it (the hybrid condensation executes ~1/6 of the survey count)
        achieved = sfl / (t_ms / 1000.0) / 1e12
        roof = {"kernel": {"band": "band_solve_kernel (Stokes: assembly + banded LU + multi-RHS)",
                           "hybrid": "condense_kernel (Darcy: SPD static condensation)"}[dom],
                "bound": "fp64 (DMMA)", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak if peak else None,
                "peak_source": "profiles/fp64_peak.json (our DMMA microbenchmark; "
                               "MEASURED_PEAKS.json has no FP64 figure)",
                "algorithmic_flops_per_launch": sfl / cnt, "executed_flops_per_launch": fl / cnt, "launch_ms": t_ms / cnt,
                "share_of_step": t_ms / tot_ms if tot_ms else None,
                "executed_tflops": fl / (t_ms / 1000.0) / 1e12,
                "executed_frac": (fl / (t_ms / 1000.0) / 1e12) / peak if peak else None,
                "traffic": _traffic(dom, a.config)[0],
                "traffic_unit": "bytes/launch (dram read + write, ncu --set full)",
                "traffic_source": _traffic(dom, a.config)[1],
                "per_kind_ms_per_step": {k: v[0] / len(dev_ms) for k, v in kinds.items()}}
        if dom == "band":
            lay = plan.problem.layout
            n_max = max([int(plan.patterns[i].n) for i in range(plan.n_sub)
                         if lay.physics(i) == "stokes"], default=0)
            roof["note"] = (f"latency bound, not throughput bound: the banded LU is a chain of "
                            f"n/16 = {(n_max + 15) // 16} dependent panel factorizations per "
                            f"system (17-18 us each on the measured timeline: factor 10.7, "
                            f"next-block update 4.1, publication 3.3), with the trailing and rhs "
                            f"updates overlapped off the chain (DESIGN.md 4.2)")
    # wall time of the basis phase (Stokes and Darcy waves run concurrently)
    basis_ms = float(np.mean(bases_ms)) if bases_ms else \
        sum(v[0] for v in kinds.values()) / max(len(dev_ms), 1)
    # batched CG: SURVEY 8(d) bytes per point-iteration 8 sum_i N_dof,i^2 + 48 n_lambda
    roof_cg = None
    if cg_ms and iters_host is not None and ws == 1:
        per_it = 8.0 * float(np.sum(plan.ndof.astype(np.int64) ** 2)) + 48.0 * nl
        t = float(np.mean(cg_ms)) / 1000.0
        ach = per_it * float(np.sum(iters_host)) / t / 1e9
        hbm = float(peaks.get("hbm_copy_gbs", peaks.get("hbm_gbs", 0.0)) or 0.0) if peaks else 0.0
        roof_cg = {"kernel": cg_name, "bound": "hbm",
                   "achieved": ach, "peak": hbm or None, "unit": "GB/s",
                   "frac": ach / hbm if hbm else None,
                   "algorithmic_bytes_per_point_iteration": per_it,
                   "point_iterations": int(np.sum(iters_host)), "launch_ms": t * 1000.0,
                   "traffic": _traffic("cg", a.config)[0],
                   "note": "algorithmic bytes as if every block were read from HBM per "
                           "point-iteration; the kernel reads them once per point"}
    # bytes of the per-step inputs run_method uploads (collocation + KL tables)
    h2d = int(res.timings.get("h2d_bytes", 0)) if (res is not None and hasattr(res, "timings")) \
        else 0
    # lambdas, residual histories (the whole [n_real, max_iter] buffer when it
    # is small -- run_method packs it on the host -- else the packed entries),
    # iters + status, moments
    n_hist = grid.n_real * max_iter
    if n_hist * 8 > (256 << 20) and iters_host is not None:
        n_hist = int(np.sum(iters_host))
    d2h = 8 * grid.n_real * nl + 8 * n_hist + 8 * grid.n_real * 2 + \
        16 * (nl + int(plan.nfield.sum()))
    if rank == 0:
        line = {
            "metric": f"collocation realizations/s (S3 sweep, {a.config})",
            "value": value, "unit": "realizations/s", "n_gpus": ws, "steps": a.steps,
            "warmup": a.warmup, "warmup_extra_steps": extra, "ms_per_step": ms_step,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (deterministic Gauss-Hermite/Smolyak collocation of the "
                    "config; no dataset)",
            "config": {"workload": a.config, "n_real": grid.n_real, "n_lambda": nl,
                       "systems": len(systems), "tol": a.tol,
                       "parallelism": (f"sharded x{ws}: subdomains (pre-loop + moments), "
                                       f"points (CG); NCCL all-reduce/all-gather")
                       if ws > 1 else "single",
                       "l2": "flushed (256 MB write) before every timed step",
                       "plan_cached": True, "plan_build_s": plan_s},
            "basis_local_solves_per_s": local_solves / (basis_ms / 1000.0) if basis_ms else None,
            "cg_iters_mean": float(iters_host.mean()), "cg_iters_max": int(iters_host.max()),
            "roofline": roof,
            "roofline_cg": roof_cg,
            "gpu_launches": launches,
            "e2e": {"value": e2e_val, "unit": "realizations/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "api": "run_method(problem, grid, 'S3', tol)"},
            "clocks": clocks.summary(),
        }
        if not a.no_s2 and ws == 1:
            line["s2_comparison"] = s2_comparison(plan, problem, grid, a.tol, max_iter, flush)
        if not a.no_s2 and ws == 1:
            hbm = float(peaks.get("hbm_copy_gbs", peaks.get("hbm_gbs", 0.0)) or 0.0) \
                if peaks else 0.0
            line["s1_comparison"] = s1_comparison(plan, problem, grid, a.tol, hbm or None)
        if not a.no_cpu_baseline and ws == 1:
            cb = cpu_baseline(cfg_path, a.tol)
            line["cpu_baseline"] = {
                "value": cb["realizations_per_s"], "unit": "realizations/s", "cores": 1,
                "kind": "port",
                "sample": f"oracle/s3_cpu.py full {a.config} S3 sweep ({cb['n_real']} points), "
                          f"1 BLAS thread",
                "basis_local_solves_per_s": cb["basis_local_solves_per_s"],
                "pre_loop_s": cb["pre_loop_s"], "main_loop_s": cb["main_loop_s"]}
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
