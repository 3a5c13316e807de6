"""CG phase cycle breakdown of the staged cg_kernel (CTA 0, -DMFB_PROFILE build
_mfb_prof.so); the register-row cg_pair_kernel has no phase hooks."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1802_06263_b200 import _lib

_lib._lib = None
_lib.load(os.path.join(os.path.dirname(_lib._SO), "_mfb_prof.so"))
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
problem, grid, _ = load_config(f"configs/{cfg}.json")
plan = get_plan(problem, grid)
eng = SweepEngine(plan)
eng.kl_fields()
eng.build_bases()
# the CGP phase hooks live in the staged one-CTA-per-point kernel (cg_kernel)
lam, iters, status, hist, _ = eng.solve_points(1e-11, 10 * plan.n_lambda, kernel="staged")
torch.cuda.synchronize()
out = (ctypes.c_ulonglong * 8)()
_lib.load().mfb_debug_cgprof(out)
v = np.array(out[:], dtype=np.float64)
it = int(iters.cpu().numpy()[0])
names = {1: "zero Sp + sync", 2: "GEMV (+pSp part)", 3: "reduce pSp", 4: "x,r update", 5: "reduce rr",
         6: "tail (sqrt, beta, p)"}
tot = sum(v[i] for i in names)
print(f"CTA 0: {it} iterations, {tot / max(it, 1):.0f} cycles/iteration")
for i, n in names.items():
    print(f"  {n:22s} {v[i] / max(it, 1):8.0f} cycles/it  {100 * v[i] / tot:5.1f}%")
