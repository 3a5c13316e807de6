"""Phase cycle breakdown of the Darcy condense kernel (CTA 0), -DMFB_PROFILE build."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1802_06263_b200 import _lib

_lib._lib = None
_lib.load(os.path.join(os.path.dirname(_lib._SO), "_mfb_prof.so"))
from paper_1802_06263_b200.config import load_config  # noqa: E402
from paper_1802_06263_b200.interface import S3Engine, get_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
problem, grid, _ = load_config(f"configs/{cfg}.json")
if cfg == "cfg5":
    from paper_1802_06263_b200.collocation import build_tensor_grid
    loc = build_tensor_grid([3] * 6)
    grid.local_points = [loc.points.copy() for _ in problem.perm.regions]
    grid.local_counts = [loc.n_real] * len(problem.perm.regions)
plan = get_plan(problem, grid)
eng = S3Engine(plan, keep_fields=(cfg != "cfg5"))
eng.kl_fields()
eng.build_bases()
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 16)()
print("rc", _lib.load().mfb_debug_prof(out))
v = np.array(out[:], dtype=np.float64)
names = {1: "copy", 5: "branch(w0 panel)", 2: "wait", 3: "sbad", 4: "store+dmma",
         13: "branch(w1 assembly)"}
tot = v[1] + v[5] + v[2] + v[3] + v[4]
for i, nme in names.items():
    print(f"{nme:22s} {v[i] / 1e6:10.3f} Mcycles  {100 * v[i] / tot:5.1f}%")
h = plan.hyb[plan.darcy[0]]
print("n", h.n, "w", h.w, "panels", (h.n + 7) // 8)

out = (ctypes.c_ulonglong * 16)()
_lib.load().mfb_debug_bprof(out)
v = np.array(out[:], dtype=np.float64)
names = {1: "load panel", 2: "panel factor", 3: "perm+writeback", 4: "phase A (stage+U12)",
         6: "phase A' (rhs top)", 8: "phase B (DMMA trailing)", 5: "phase B' (rhs below)",
         7: "back substitution"}
tot = sum(v[i] for i in names)
print("band_solve CTA 0 (first Stokes system):")
for i, nme in names.items():
    print(f"  {nme:30s} {v[i] / 1e6:10.3f} Mcycles  {100 * v[i] / tot:5.1f}%")
