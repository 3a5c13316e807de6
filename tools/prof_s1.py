"""One Method-S1 sweep of a config (for ncu captures of band_apply_kernel /
s1_cg_step_kernel): python tools/prof_s1.py [cfg] [max_iter]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 64
problem, grid, _ = load_config(os.path.join("configs", f"{name}.json"))
plan = get_plan(problem, grid)
eng = SweepEngine(plan, method="S2", darcy_kernel="band", keep_factors=True)
eng.kl_fields()
eng.build_bases()
eng.solve_s1(1e-11, max_iter)
eng.torch.cuda.synchronize()
print("ok", eng.launches)
