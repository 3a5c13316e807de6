"""Check and time the cluster CG (mfb_cg_cluster) against the 8-points-per-CTA
kernel: cfg2 parity vs the reference golden per shape (lambda, iterations,
point-alone bitwise), then a cfg4 slice (n_pts points x iters iterations,
points end in MAX_ITER) per kernel.

usage: python tools/prof_cg_cluster.py [n_pts] [iters] [shapes e.g. 4x16,8x16] [--no-check]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
n_pts = int(args[0]) if len(args) > 0 else 2368
iters = int(args[1]) if len(args) > 1 else 200
shapes = ([tuple(int(v) for v in s.split("x")) for s in args[2].split(",")] if len(args) > 2
          else [(4, 16), (8, 16), (2, 8), (4, 8)])


def hist_rows(hist, it):
    if hasattr(hist, "to_host"):
        return hist.to_host(it)
    h = hist.cpu().numpy()
    return [h[k, :it[k]] for k in range(len(it))]


if "--no-check" not in sys.argv:
    from conftest import case_from_golden
    z = np.load(os.path.join(ROOT, "tests", "golden", "cfg2.npz"))
    _, problem, grid, _ = case_from_golden("cfg2")
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, keep_fields=False)
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    max_iter = max(50, 10 * plan.n_lambda)
    ref = z["s3_lambda"]
    for shp in shapes:
        lam, it, st, hist, g = eng.solve_points(1e-11, max_iter, keep_g=True, kernel="cluster",
                                                cluster_shape=[shp])
        torch.cuda.synchronize()
        L = lam.cpu().numpy()[z["s3_points"]]
        itn = it.cpu().numpy()
        err = np.linalg.norm(L - ref) / np.linalg.norm(ref)
        gerr = np.max(np.abs(g.cpu().numpy()[z["s3_points"]] - z["s3_g"])) / np.max(np.abs(z["s3_g"]))
        H = hist_rows(hist, itn)
        last_ok = all(H[k][-1] <= 1e-11 for k in range(len(itn)))
        k = 54
        lam1, it1, _, _, _ = eng.solve_points(1e-11, max_iter, k0=k, n_pts=1, kernel="cluster",
                                              cluster_shape=[shp])
        alone = (np.array_equal(lam1.cpu().numpy()[0], lam.cpu().numpy()[k])
                 and int(it1.cpu()[0]) == int(itn[k]))
        print(f"cfg2 cluster {shp}: {eng.cg_kernel_name}: lambda rel {err:.2e}, g {gerr:.1e}, "
              f"status {np.bincount(st.cpu().numpy())}, iters mean {itn.mean():.1f} "
              f"(ref {z['s3_iters'].mean():.1f}), hist last<=tol {last_ok}, alone bitwise {alone}",
              flush=True)

problem, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields()
eng.build_bases()
torch.cuda.synchronize()
nd2 = float(np.sum(plan.ndof.astype(np.int64) ** 2))
runs = [("multi", None)] + [("cluster", s) for s in shapes]
base = None
for kern, shp in runs:
    for rep in range(2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lam, it, st, hist, _ = eng.solve_points(1e-30, iters, k0=0, n_pts=n_pts,
                                                kernel=kern,
                                                cluster_shape=[shp] if shp else None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        pi = float(it.sum().item())
        L = lam.cpu().numpy()
        if base is None:
            base = L
        dev = np.max(np.abs(L - base)) / np.max(np.abs(base))
        print(f"cfg4 {kern} {shp or ''} rep {rep}: {n_pts} x {iters} its: {ms:.1f} ms, "
              f"{1e3 * ms / pi:.4f} us/point-it, FP64 {2 * nd2 * pi / (ms / 1e3) / 1e12:.2f} "
              f"TFLOP/s (2 sum N^2), max dev vs multi {dev:.1e}", flush=True)
