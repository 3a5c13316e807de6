"""Time (and, under ncu, profile) the CG kernels on a cfg4 slice: n_pts points
for a fixed iteration budget (points end in MAX_ITER; time per iteration is
what is measured).

usage: python tools/prof_cg_multi.py [n_pts] [iters] [kernel: multi|cta|both|ab] [stride]

stride > 1: the slice is every stride-th point of the grid (a sub-grid like
bench.py's batches) instead of the first n_pts. "ab": the multi kernel with
and without the reflection-family order / chunked claims, alternating, and a
bitwise comparison of the two results; "abs": the same for the streamed S p
against the task loop. iters = 0: the real solve (tol 1e-11,
max_iter 200,000) instead of a fixed iteration budget.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200 import interface  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 1184
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
which = sys.argv[3] if len(sys.argv) > 3 else "both"
stride = int(sys.argv[4]) if len(sys.argv) > 4 else 1
problem, grid, _ = load_config("configs/cfg4.json")
if stride > 1:
    from sdmortar.collocation import CollocationGrid
    pts = np.arange(0, grid.n_real, stride)[:n_pts]
    n_pts = len(pts)
    grid = CollocationGrid(grid.kind, grid.points[pts], grid.weights[pts], grid.splits,
                           [li[pts] for li in grid.local_indices],
                           list(grid.local_counts), list(grid.local_points))
if os.environ.get("MFB_TAIL"):
    interface.MULTI_TAIL = int(os.environ["MFB_TAIL"])
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields()
eng.build_bases()
torch.cuda.synchronize()
per_it = 8.0 * float(np.sum(plan.ndof.astype(np.int64) ** 2)) + 48.0 * plan.n_lambda
runs = {"both": [("multi", None), ("cta", None)], "ab": [("multi", True), ("multi", False)] * 2,
        "abs": [("multi", True), ("multi", False)] * 2}.get(which, [(which, None)])
flag = "MULTI_STREAM" if which == "abs" else "MULTI_CHUNKS"
keep = {}
for kern, chunks in runs:
    if chunks is not None:
        setattr(interface, flag, chunks)
    for rep in range(2 if chunks is None else 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lam, it, st, h, _ = eng.solve_points(1e-30 if iters else 1e-11, iters or 200000, k0=0,
                                            n_pts=n_pts, hist_cap=iters or None, kernel=kern)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pi = float(it.sum().item())
        tag = "" if chunks is None else f" {flag}={chunks}"
        print(f"{kern}{tag} rep {rep}: {n_pts} points x {iters} its: {ms:.1f} ms, "
              f"{1e6 * ms / 1e3 / pi:.4f} us per point-iteration, algorithmic "
              f"{per_it * pi / (ms / 1e3) / 1e12:.1f} TB/s, statuses {np.bincount(st.cpu().numpy())}",
              flush=True)
        if chunks is not None:
            if chunks in keep:
                assert torch.equal(keep[chunks], lam), "rerun differs"
            keep[chunks] = lam
if len(keep) == 2:
    same = torch.equal(keep[True], keep[False])
    rel = float((keep[True] - keep[False]).abs().max() / keep[False].abs().max())
    print(f"{flag} on == off bitwise: {same}, max |diff| / max |lambda| = {rel:.2e}", flush=True)
    # (the 16-row tasks of the streamed kernel add p . S p in another order:
    # roundoff that an unconverged CG amplifies -- compare converged solves,
    # iters = 0, or a handful of iterations)
    assert same or (flag == "MULTI_STREAM" and (iters > 5 or rel < 1e-6))
