"""Per-phase device timing of one S3 (or S2) sweep (CUDA events on the launch stream).

usage: python tools/phase_timing.py cfg2 [--reps 2] [--method S2]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_1802_06263_b200.adapter import load_config
from paper_1802_06263_b200.interface import SweepEngine, get_plan


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--tol", type=float, default=1e-11)
    ap.add_argument("--no-cg", action="store_true")
    ap.add_argument("--darcy", default="hybrid", choices=["hybrid", "band"])
    ap.add_argument("--method", default="S3", choices=["S3", "S2"])
    a = ap.parse_args()
    path = a.config if a.config.endswith(".json") else f"configs/{a.config}.json"
    t = time.time()
    problem, grid, _ = load_config(path)
    t_setup = time.time() - t
    t = time.time()
    plan = get_plan(problem, grid)
    t_plan = time.time() - t
    print(f"setup {t_setup:.2f}s plan {t_plan:.2f}s n_real {grid.n_real} "
          f"n_lambda {plan.n_lambda} method {a.method}", flush=True)
    for rep in range(a.reps):
        eng = SweepEngine(plan, darcy_kernel=a.darcy, method=a.method)
        eng.timing = True
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        ev[0].record()
        eng.kl_fields()
        ev[1].record()
        eng.build_bases()
        ev[2].record()
        if not a.no_cg:
            lam, iters, status, hist, _ = eng.solve_points(a.tol, max(50, 10 * plan.n_lambda))
        ev[3].record()
        if not a.no_cg:
            eng.moments(lam)
        ev[4].record()
        torch.cuda.synchronize()
        eng.check_info()
        names = ["kl", "bases", "cg", "moments"]
        tt = [ev[i].elapsed_time(ev[i + 1]) for i in range(4)]
        msg = " ".join(f"{n} {x:.2f}ms" for n, x in zip(names, tt))
        if not a.no_cg:
            it = iters.cpu().numpy()
            msg += f" | iters mean {it.mean():.1f} max {it.max()} status {np.bincount(status.cpu().numpy())}"
        print(f"rep {rep}: {msg}", flush=True)
        for kind, a0, a1, fl, sfl in eng.solve_events:
            ms = a0.elapsed_time(a1)
            print(f"   {kind:6s} launch {ms:8.2f} ms, {fl / 1e9:8.2f} GFLOP executed "
                  f"({fl / ms / 1e9:6.2f} TF/s), survey-algorithmic {sfl / 1e9:8.2f} GFLOP "
                  f"({sfl / ms / 1e9:6.2f} TF/s)")


if __name__ == "__main__":
    main()
