"""Per-iteration time of Method S1's CG vs the number of live points (cfg2):
one event per iteration around apply + step. python tools/s1_iter_profile.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200 import _lib  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

problem, grid, _ = load_config(os.path.join("configs", "cfg2.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, method="S2", darcy_kernel="band", keep_factors=True)
eng.kl_fields()
eng.build_bases()
lam, iters, status, hist, _ = eng.solve_s1(1e-11, 2000)     # warm
torch.cuda.synchronize()
it = np.sort(iters.cpu().numpy())
# time the same solve in slices of 50 iterations: the live count at iteration
# j is the number of points with iters >= j
orig = eng._s1_apply
evs = []


def timed_apply(*a, **k):
    e = torch.cuda.Event(enable_timing=True)
    e.record(eng.stream)
    evs.append(e)
    return orig(*a, **k)


eng._s1_apply = timed_apply
eng.solve_s1(1e-11, 2000, check_every=16)
torch.cuda.synchronize()
ms = np.array([evs[j].elapsed_time(evs[j + 1]) for j in range(len(evs) - 1)])
for j0 in range(0, min(len(ms), int(it.max()) + 1), 100):
    live = int(np.sum(it > j0))
    print(f"iterations {j0:5d}-{j0 + 99:5d}: live points {live:4d}, "
          f"{ms[j0:j0 + 100].mean():.3f} ms per iteration", flush=True)
print("total", ms.sum())
