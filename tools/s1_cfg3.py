"""Method S1 on cfg3 (609 realizations, factors ~1 TB in total): runs in
realization chunks. python tools/s1_cfg3.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import run_method  # noqa: E402

problem, grid, _ = load_config(os.path.join("configs", "cfg3.json"))
t0 = time.perf_counter()
res = run_method(problem, grid, method="S1", tol=1e-11)
wall = time.perf_counter() - t0
it = np.array(res.stats.cg_iters)
print(f"cfg3 S1: {grid.n_real} points in {res.timings['chunks']} chunks, iters mean "
      f"{it.mean():.0f} max {it.max()}, wall {wall:.1f} s ({grid.n_real / wall:.2f} "
      f"realizations/s)", flush=True)
r3 = run_method(problem, grid, method="S3", tol=1e-11)
L1, L3 = np.array(res.lambdas), np.array(r3.lambdas)
print("S1 vs S3 lambda rel diff (different methods: S3 freezes Stokes at the mean)",
      float(np.linalg.norm(L1 - L3) / np.linalg.norm(L3)))
