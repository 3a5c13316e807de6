"""Method S1 sweep timing on the device (second run timed; the first builds
the plan and the sweep state): python tools/s1_timing.py [cfg ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import run_method  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    problem, grid, _ = load_config(os.path.join("configs", f"{name}.json"))
    for rep in range(2):
        t0 = time.perf_counter()
        res = run_method(problem, grid, method="S1", tol=1e-11)
        wall = time.perf_counter() - t0
    it = np.array(res.stats.cg_iters)
    tm = res.timings
    print(f"{name} S1: {grid.n_real} points, iters mean {it.mean():.0f} max {it.max()}, "
          f"wall {wall * 1e3:.1f} ms ({grid.n_real / wall:.1f} realizations/s), "
          f"bases {tm['bases'] * 1e3:.1f} ms, cg {tm['cg'] * 1e3:.1f} ms, "
          f"recovery+moments {tm['moments'] * 1e3:.1f} ms", flush=True)
