"""cProfile of one warm run_method call on a cfg4 bench batch (host-side costs
of the end-to-end path: staging, verdict checks, residual histories, moments).

usage: python tools/prof_e2e_cfg4.py [batches]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import run_method  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4
problem, grid, opts = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
g = bench._batch_grids(grid, B)[0]
mi = opts.get("max_iter")
kw = dict(tol=1e-11, max_iter=mi or 200000)
t0 = time.perf_counter()
res = run_method(problem, g, "S3", **kw)
torch.cuda.synchronize()
print(f"cold call {time.perf_counter() - t0:.2f} s", flush=True)
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
res = run_method(problem, g, "S3", **kw)
pr.disable()
wall = time.perf_counter() - t0
tm = getattr(res, "timings", None)
print(f"warm call {wall:.2f} s; timings {tm}", flush=True)
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
