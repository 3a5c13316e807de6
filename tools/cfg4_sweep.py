"""Full cfg4 Method S3 sweep on the device through run_method (54,273 points,
n_lambda = 2,720), with per-phase wall times, CG iteration statistics and, when
tests/golden/cfg4_points.npz is present, lambda parity on its sampled points.

usage: python tools/cfg4_sweep.py [--tol 1e-11] [--json out.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import run_method  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tol", type=float, default=1e-11)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--json", default=None)
    ap.add_argument("--max-iter", type=int, default=None,
                    help="CG iteration cap (reference default max(50, 10 n_lambda))")
    a = ap.parse_args()
    t = time.time()
    problem, grid, _ = load_config(os.path.join(ROOT, "configs", f"{a.config}.json"))
    setup_s = time.time() - t
    torch.cuda.synchronize()
    t = time.time()
    res = run_method(problem, grid, method="S3", tol=a.tol, max_iter=a.max_iter,
                     basis_cap_mb=1e6)
    torch.cuda.synchronize()
    wall = time.time() - t
    it = np.asarray(res.stats.cg_iters)
    out = {"config": a.config, "n_real": int(grid.n_real), "n_lambda": int(problem.space.n_dof),
           "tol": a.tol, "max_iter": a.max_iter, "setup_s": setup_s, "run_method_s": wall,
           "realizations_per_s": grid.n_real / wall,
           "timings": {k: float(v) for k, v in res.timings.items()},
           "cg_iters_mean": float(it.mean()), "cg_iters_max": int(it.max()),
           "cg_iters_min": int(it.min()), "point_iterations": int(it.sum()),
           "cg_iters_percentiles": {q: int(np.percentile(it, q)) for q in (50, 90, 99, 99.9)},
           "slowest_points": [int(k) for k in np.argsort(it)[-5:]],
           "residual_entries": int(len(res.residuals.flat))
           if hasattr(res.residuals, "flat") else None}
    gold = os.path.join(ROOT, "tests", "golden", f"{a.config}_points.npz")
    if os.path.exists(gold):
        z = np.load(gold)
        errs = {}
        for j, k in enumerate(z["points"]):
            ref = z["lambda"][j]
            errs[int(k)] = {"lambda_rel": float(np.linalg.norm(res.lambdas[k] - ref)
                                                / np.linalg.norm(ref)),
                            "iters": int(it[k]), "iters_ref": int(z["iters"][j])}
        out["golden_points"] = errs
    mk = res.moments
    out["moment_keys"] = len(mk)
    out["lambda_mean_norm"] = float(np.linalg.norm(mk["lambda"][0]))
    out["lambda_var_norm"] = float(np.linalg.norm(mk["lambda"][1]))
    print(json.dumps(out, indent=1), flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(out, f, indent=1)
        np.savez_compressed(a.json.replace(".json", "_moments.npz"),
                            **{k.replace(":", "_") + "_mean": v[0] for k, v in mk.items()},
                            **{k.replace(":", "_") + "_var": v[1] for k, v in mk.items()})


if __name__ == "__main__":
    main()
