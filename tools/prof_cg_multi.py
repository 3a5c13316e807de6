"""Time (and, under ncu, profile) the CG kernels on a cfg4 slice: n_pts points
for a fixed iteration budget (points end in MAX_ITER; time per iteration is
what is measured).

usage: python tools/prof_cg_multi.py [n_pts] [iters] [kernel: multi|cta|both]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
which = sys.argv[3] if len(sys.argv) > 3 else "both"
problem, grid, _ = load_config("configs/cfg4.json")
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields()
eng.build_bases()
torch.cuda.synchronize()
per_it = 8.0 * float(np.sum(plan.ndof.astype(np.int64) ** 2)) + 48.0 * plan.n_lambda
for kern in (["multi", "cta"] if which == "both" else [which]):
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lam, it, st, h, _ = eng.solve_points(1e-30, iters, k0=0, n_pts=n_pts, hist_cap=iters,
                                            kernel=kern)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pi = float(it.sum().item())
        print(f"{kern} rep {rep}: {n_pts} points x {iters} its: {ms:.1f} ms, "
              f"{1e6 * ms / 1e3 / pi:.3f} us per point-iteration, algorithmic "
              f"{per_it * pi / (ms / 1e3) / 1e12:.1f} TB/s, statuses {np.bincount(st.cpu().numpy())}",
              flush=True)
