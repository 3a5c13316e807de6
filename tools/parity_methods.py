"""Parity of the device Methods S2 and S1 vs the reference's own S2 / S1
sweeps (tests/golden/*_s2.npz, *_s1.npz) -> JSON.

usage: python tools/parity_methods.py > profiles/rNN/parity_methods.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from conftest import GOLDEN, case_from_golden  # noqa: E402
from paper_1802_06263_b200.interface import run_method  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / max(np.linalg.norm(np.ravel(b)), 1e-300))


out = []
for method, tag in (("S2", "s2"), ("S1", "s1")):
    for name in ("cfg1", "darcy_twoblock", "case1_mini", "cfg2"):
        path = os.path.join(GOLDEN, f"{name}_{tag}.npz")
        if not os.path.exists(path):
            continue
        z = np.load(path)
        _, problem, grid, _ = case_from_golden(name)
        res = run_method(problem, grid, method=method, tol=1e-11)
        keys = [k for k in res.moments if k != "lambda"]
        mean_err = {k: rel(res.moments[k][0], z[f"mean__{k}"]) for k in keys}
        var_err = {k: rel(res.moments[k][1], z[f"var__{k}"]) for k in keys}
        wm, wv = max(mean_err, key=mean_err.get), max(var_err, key=var_err.get)
        it = np.array(res.stats.cg_iters)
        out.append({"method": method, "config": name, "n_real": grid.n_real,
                    "lambda_rel_err": rel(np.array(res.lambdas), z[f"{tag}_lambda"]),
                    "lambda_mean_rel_err": rel(res.moments["lambda"][0], z["mean__lambda"]),
                    "field_mean_worst": [wm, mean_err[wm]], "field_var_worst": [wv, var_err[wv]],
                    "iters_mean": float(it.mean()), "iters_mean_ref": float(z[f"{tag}_iters"].mean()),
                    "backsolves_equal_ref": bool(np.array_equal(res.stats.backsolves,
                                                                z["stats_backsolves"]))})
print(json.dumps(out, indent=1))
