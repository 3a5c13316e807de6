"""Per-phase clock breakdown of the cluster CG (debug build path:
mfb_debug_cluster(100) records clock64 deltas at the phase boundaries in
thread 0 of every CTA) on a cfg4 slice.

usage: python tools/cluster_phases.py [n_pts] [iters] [CxNP ...]
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200 import _lib  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 2112
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
shapes = [tuple(int(v) for v in a.split("x")) for a in sys.argv[3:]] or [(4, 16)]
problem, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields()
eng.build_bases()
L = _lib.load()
names = ["refill+run", "phaseA(w0)", "wait#1", "A2+pSp", "phaseB+rr", "phaseC", "wait#4"]
for shp in shapes:
    eng.solve_points(1e-30, iters, n_pts=n_pts, kernel="cluster", cluster_shape=[shp])
    torch.cuda.synchronize()
    L.mfb_debug_cluster(100)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, it, _, _, _ = eng.solve_points(1e-30, iters, n_pts=n_pts, kernel="cluster",
                                      cluster_shape=[shp])
    e1.record()
    torch.cuda.synchronize()
    L.mfb_debug_cluster(0)
    ct = eng.st._cluster[shp]
    n_cta = ct["n_clusters"] * shp[0]
    buf = (ctypes.c_longlong * (8 * 1024))()
    L.mfb_debug_cluster_prof(buf, 8 * 1024)
    full = np.array(buf[:], dtype=np.float64)
    a = full[:8 * n_cta].reshape(n_cta, 8)
    w = full[4 * 1024:4 * 1024 + 4 * n_cta].reshape(n_cta, 4) / np.maximum(a[:, 7:8], 1)
    print(f"  per CTA-iteration: strips {w[:, 0].mean():.0f}, fragments {w[:, 1].mean():.0f}, "
          f"MMA half0 frags {w[:, 2].mean():.0f}, half1 frags {w[:, 3].mean():.0f}", flush=True)
    its = a[:, 7].mean()
    per = a[:, :7].sum(0) / max(a[:, 7].sum(), 1)
    print(f"{shp}: {e0.elapsed_time(e1):.1f} ms, {its:.0f} iterations per CTA, cycles per "
          f"iteration {per.sum():.0f} = " + ", ".join(f"{n} {v:.0f}" for n, v in zip(names, per)),
          flush=True)
