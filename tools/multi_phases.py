"""Per-phase clock breakdown of the multi-point CG (mfb_debug_multi) on a cfg4
slice: refill, S p (warp 0), reduce #1, update x/r, reduce #2, p update.

usage: python tools/multi_phases.py [n_pts] [iters]
"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1802_06263_b200 import _lib, interface
interface.MULTI_CHUNKS = os.environ.get("MFB_CHUNKS", "1") == "1"
interface.MULTI_STREAM = os.environ.get("MFB_STREAM", "1") == "1"
from paper_1802_06263_b200.adapter import load_config
from paper_1802_06263_b200.interface import SweepEngine, get_plan
n_pts = int(sys.argv[1]) if len(sys.argv) > 1 else 2368
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
problem, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields(); eng.build_bases()
L = _lib.load()
eng.solve_points(1e-30, iters, n_pts=n_pts, kernel="multi")
torch.cuda.synchronize()
L.mfb_debug_multi(1, None)
L.mfb_debug_multi_warps(None, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
_, it, _, _, _ = eng.solve_points(1e-30, iters, n_pts=n_pts, kernel="multi")
e1.record()
torch.cuda.synchronize()
L.mfb_debug_multi(0, None)
buf = (ctypes.c_longlong * (148 * 8))()
L.mfb_debug_multi(0, buf)
a = np.array(buf[:], dtype=np.float64).reshape(148, 8)
per = a[:, :6].sum(0) / max(a[:, 6].sum(), 1)
names = ["refill", "S p (warp 0)", "reduce#1", "x,r update", "reduce#2", "p update+fin"]
print(f"list_cap {eng.st._multi['list_cap']} stream {interface.MULTI_STREAM}: {e0.elapsed_time(e1):.1f} ms, {a[:, 6].mean():.0f} iterations per CTA, cycles per "
      f"iteration {per.sum():.0f} = " + ", ".join(f"{n} {v:.0f}" for n, v in zip(names, per)))

wb = (ctypes.c_longlong * 16)()
L.mfb_debug_multi_warps(wb, 0)
w = np.array(wb[:], dtype=np.float64) / max(a[0, 6], 1)
h = eng.st._multi
tab = None
print("S p cycles per iteration by warp of CTA 0:", " ".join(f"{v:.0f}" for v in w))
