"""Phase cycle breakdown of the Darcy condense kernel (CTA 0), -DMFB_PROFILE build."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1802_06263_b200 import _lib

_lib._lib = None
_lib.load(os.environ.get("MFB_PROF_LIBRARY") or os.path.join(os.path.dirname(_lib._SO), "_mfb_prof.so"))
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
band_only = "--band" in sys.argv
problem, grid, _ = load_config(f"configs/{cfg}.json")
if cfg == "cfg5":
    from sdmortar.collocation import build_tensor_grid
    loc = build_tensor_grid([3] * 6)
    grid.local_points = [loc.points.copy() for _ in problem.perm.regions]
    grid.local_counts = [loc.n_real] * len(problem.perm.regions)
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=(cfg != "cfg5"))
eng.kl_fields()
eng.build_bases()
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 16)()
print("rc", _lib.load().mfb_debug_prof(out))
v = np.array(out[:], dtype=np.float64)
names = {1: "copy", 5: "branch(w0 panel)", 2: "wait", 3: "sbad", 4: "store+dmma",
         13: "branch(w1 assembly)", 14: "  w1: zero + bar", 15: "  w1: entries"}
tot = v[1] + v[5] + v[2] + v[3] + v[4]
for i, nme in names.items():
    print(f"{nme:22s} {v[i] / 1e6:10.3f} Mcycles  {100 * v[i] / tot:5.1f}%")
h = plan.hyb[plan.darcy[0]]
print("n", h.n, "w", h.w, "panels", (h.n + 7) // 8)

out = (ctypes.c_ulonglong * 24)()
_lib.load().mfb_debug_bprof(out)
v = np.array(out[:], dtype=np.float64)
names = {1: "wait + load panel k", 2: "update block k+1 (owner)", 3: "factor panel k+1 (owner)",
         4: "update other blocks", 5: "rhs forward + DMMA", 0: "loop head", 7: "back substitution",
         8: "  upd: stage rows", 9: "  upd: moved rows", 10: "  upd: U12 forward", 11: "  upd: DMMA", 12: "  fac: load", 13: "  fac: columns", 14: "  fac: publish",
         15: "  fac: fence+release", 17: "  bs: issue U loads", 18: "  bs: window+U11 prefetch",
         19: "  bs: solve", 20: "  bs: push"}
tot = sum(v[i] for i in names)
print("band_solve CTA 0 (first Stokes system):")
for i, nme in names.items():
    print(f"  {nme:30s} {v[i] / 1e6:10.3f} Mcycles  {100 * v[i] / tot:5.1f}%")

if band_only or True:
    tl = (ctypes.c_ulonglong * (4 * 4096))()
    if _lib.load().mfb_debug_timeline(tl) == 0:
        t = np.array(tl[:], dtype=np.float64).reshape(4, 4096)
        pats = [p for p in plan.patterns if p.nb >= 0]
        nb = None
        for s_, p_ in enumerate(plan.patterns):
            if s_ not in plan.hyb:
                nb = (p_.n + 15) // 16
                break
        if nb:
            m = nb - 1
            arrive, start, upd, pub = t[3, :m], t[0, :m], t[1, :m], t[2, :m]
            ok = (arrive > 0) & (start > 0) & (pub > 0)
            print("system-0 panel chain (us, median over %d panels):" % ok.sum())
            print("  owner arrives at wait -> sees panel k   %8.2f" % np.median((start - arrive)[ok] / 1e3))
            print("  update block k+1                        %8.2f" % np.median((upd - start)[ok] / 1e3))
            print("  factor + publish k+1                    %8.2f" % np.median((pub - upd)[ok] / 1e3))
            nxt = start[1:] - pub[:-1]
            ok2 = ok[1:] & ok[:-1]
            print("  publish k -> owner of k+1 sees it       %8.2f" % np.median(nxt[ok2] / 1e3))
            late = arrive[1:] - pub[:-1]
            print("  owner of k+1 arrives after publish k by %8.2f (median; >0 = late)" % np.median(late[ok2] / 1e3))
            print("  panel period                            %8.2f" % np.median(np.diff(pub[ok]) / 1e3))
