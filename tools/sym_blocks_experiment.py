import os, sys
ROOT = "/root/repo"
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from conftest import case_from_golden
from paper_1802_06263_b200.interface import SweepEngine, get_plan
for name in ["cfg2", "cfg3"]:
    z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    _, problem, grid, _ = case_from_golden(name)
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, keep_fields=False)
    eng.kl_fields(); eng.build_bases(); eng.check_info()
    mi = max(50, 10 * plan.n_lambda)
    lam, it, st, h, _ = eng.solve_points(1e-11, mi)
    ref = z["s3_iters"]
    print(name, "device mean", it.float().mean().item(), "ref", ref.mean())
    # asymmetry of device blocks per physics
    stt = eng.st
    blocks = stt.blocks
    asym = {"stokes": 0.0, "darcy": 0.0}
    for s in range(plan.n_sub):
        nd = int(plan.ndof[s]); nloc = int(stt.n_loc[s]); off = int(stt.blk_base[s])
        B = blocks[off:off + nloc * nd * nd].view(nloc, nd, nd)
        a = ((B - B.transpose(1, 2)).abs().amax() / B.abs().amax()).item()
        key = "darcy" if plan.region[s] >= 0 else "stokes"
        asym[key] = max(asym[key], a)
        if key == "stokes":
            B.copy_(0.5 * (B + B.transpose(1, 2)))
    print(name, "asymmetry", asym)
    lam2, it2, st2, h2, _ = eng.solve_points(1e-11, mi)
    print(name, "after symmetrizing Stokes blocks: mean", it2.float().mean().item(), "lambda rel change", ((lam2 - lam).norm() / lam.norm()).item())
    for s in range(plan.n_sub):
        nd = int(plan.ndof[s]); nloc = int(stt.n_loc[s]); off = int(stt.blk_base[s])
        B = blocks[off:off + nloc * nd * nd].view(nloc, nd, nd)
        B.copy_(0.5 * (B + B.transpose(1, 2)))
    lam3, it3, _, _, _ = eng.solve_points(1e-11, mi)
    print(name, "after symmetrizing all blocks: mean", it3.float().mean().item())
