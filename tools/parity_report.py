"""Parity of the device S3 path vs the reference goldens, per config -> JSON.

usage: python tools/parity_report.py [cfg1 cfg2 ...] > profiles/rNN/parity.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from conftest import case_from_golden, golden  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan, run_method  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


def report(name):
    z = golden(name)
    _, problem, grid, _ = case_from_golden(name)
    out = {"config": name, "n_real": grid.n_real, "n_lambda": problem.space.n_dof}
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan)
    eng.kl_fields()
    eng.build_bases()
    blocks = eng.blocks.cpu().numpy()
    errs = []
    by_phys = {"darcy": 0.0, "stokes": 0.0}
    for idx, (s, l) in enumerate(eng.systems):
        key = f"B__{s}__{l}"
        if key in z:
            nd = int(plan.ndof[s])
            B = blocks[eng.sys_boff[idx]: eng.sys_boff[idx] + nd * nd].reshape(nd, nd).T
            e = float(np.max(np.abs(B - z[key])) / np.max(np.abs(z[key])))
            errs.append(e)
            ph = problem.layout.physics(s)
            by_phys[ph] = max(by_phys[ph], e)
    out["basis_max_rel_err_by_physics"] = by_phys
    out["basis_blocks_checked"] = len(errs)
    out["basis_max_rel_err"] = max(errs) if errs else None
    if "s3_lambda" in z:
        res = run_method(problem, grid, method="S3", tol=1e-11)
        L = np.array(res.lambdas)[z["s3_points"]]
        out["lambda_rel_err"] = rel(L, z["s3_lambda"])
        out["lambda_ref_floor"] = float(z["floor_lambda"])
        worst_m = worst_v = worst_vm2 = 0.0
        worst_key = None
        vf = {}
        for key, (m, v) in res.moments.items():
            if f"mean__{key}" not in z:
                continue
            mg, vg = z[f"mean__{key}"], z[f"var__{key}"]
            worst_m = max(worst_m, rel(m, mg))
            rv = rel(v, vg)
            if rv > worst_v:
                worst_v, worst_key = rv, key
            worst_vm2 = max(worst_vm2, float(np.max(np.abs(v - vg)) / max(np.max(mg * mg), 1e-300)))
            vf[key] = (rv, float(z[f"floor_var__{key}"]))
        out["mean_worst_rel_err"] = worst_m
        out["var_worst_rel_err"] = worst_v
        out["var_worst_key"] = worst_key
        out["var_worst_key_ref_floor"] = vf[worst_key][1] if worst_key else None
        out["var_max_abs_over_max_mean2"] = worst_vm2
        out["iters_mean"] = float(np.mean(res.stats.cg_iters))
        out["iters_mean_ref"] = float(np.mean(z["s3_iters"]))
    return out


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg1", "darcy_twoblock", "case1_mini", "cfg2", "cfg3"]
    print(json.dumps([report(n) for n in names], indent=1))
