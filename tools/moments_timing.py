"""Host/device split of SweepEngine.moments (debug helper)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1802_06263_b200 import interface  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
problem, grid, _ = load_config(f"configs/{cfg}.json")
plan = get_plan(problem, grid)
eng = SweepEngine(plan)
eng.kl_fields()
eng.build_bases()
lam, iters, status, hist, _ = eng.solve_points(1e-11, 10 * plan.n_lambda)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    out = eng.moments(lam)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    print(f"moments total {1e3 * (t1 - t0):.2f} ms, keys {len(out)}")
import cProfile  # noqa: E402
import pstats  # noqa: E402
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    eng.moments(lam)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(14)
