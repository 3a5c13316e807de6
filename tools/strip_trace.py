"""Per-strip clock trace of warp 0, CTA 0 of the cluster CG (debug 101)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1802_06263_b200 import _lib
from paper_1802_06263_b200.adapter import load_config
from paper_1802_06263_b200.interface import SweepEngine, get_plan
shp = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "1x8").split("x"))
problem, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields(); eng.build_bases()
L = _lib.load()
eng.solve_points(1e-30, 20, n_pts=2368, kernel="cluster", cluster_shape=[shp])
torch.cuda.synchronize()
L.mfb_debug_cluster(int(os.environ.get('TRACE', '101')))
eng.solve_points(1e-30, 20, n_pts=2368, kernel="cluster", cluster_shape=[shp])
torch.cuda.synchronize()
L.mfb_debug_cluster(0)
buf = (ctypes.c_longlong * 8192)()
L.mfb_debug_cluster_prof(buf, 8192)
a = np.array(buf[:1536]).reshape(256, 6)
for i in range(0, 100):
    print(f"item {i:3d}: fill {a[i,0]:6d} take(wait) {a[i,1]:6d} mma {a[i,2]:6d}  nt4 {a[i,3]:2d} members {a[i,4]:2d} hm {a[i,5]}")
print("means: fill %.0f take %.0f mma %.0f" % (a[:100,0].mean(), a[:100,1].mean(), a[:100,2].mean()))
