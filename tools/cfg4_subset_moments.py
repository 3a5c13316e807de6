"""cfg4 subset sweep (the points of tests/golden/cfg4_moments.npz) through
run_method; per-key mean/var errors against the reference golden -> JSON.

usage: python tools/cfg4_subset_moments.py [out.json]
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1802_06263_b200.adapter import load_config
import paper_1802_06263_b200._ref  # noqa: E402,F401  (puts sdmortar on the path)
from sdmortar.collocation import CollocationGrid
from paper_1802_06263_b200.interface import run_method
z = np.load(os.path.join(ROOT, "tests", "golden", "cfg4_moments.npz"))
problem, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
pts = z["points"]
sub = CollocationGrid(grid.kind, grid.points[pts], grid.weights[pts], grid.splits,
                      [li[pts] for li in grid.local_indices], list(grid.local_counts),
                      list(grid.local_points))
res = run_method(problem, sub, method="S3", tol=float(z["tol"]), max_iter=int(z["max_iter"]),
                 basis_cap_mb=1e6)
L = np.array(res.lambdas)
out = {"lambda_rel_max": float(np.max(np.linalg.norm(L - z["lambda"], axis=1)
                                      / np.linalg.norm(z["lambda"], axis=1))),
       "iters_mean": float(np.mean(res.stats.cg_iters)), "iters_ref_mean": float(z["iters"].mean()),
       "sum_w": float(np.sum(sub.weights)), "keys": {}}
for key in [str(k) for k in z["keys"]]:
    m, v = res.moments[key]
    d = {"floor_mean": float(z[f"floor_mean__{key}"]), "floor_var": float(z[f"floor_var__{key}"])}
    if f"mean__{key}" in z.files:
        mr, vr = z[f"mean__{key}"], z[f"var__{key}"]
        d["mean_rel"] = float(np.linalg.norm(m - mr) / max(np.linalg.norm(mr), 1e-300))
        d["var_rel"] = float(np.linalg.norm(v - vr) / max(np.linalg.norm(vr), 1e-300))
        d["var_maxabs_rel"] = float(np.max(np.abs(v - vr)) / max(np.max(np.abs(vr)), 1e-300))
        d["n_var_zero_ref"] = int(np.sum(vr == 0)); d["n_var_zero_ours"] = int(np.sum(v == 0))
    else:
        idx = z[f"idx__{key}"]
        d["mean_rel"] = float(np.max(np.abs(m.reshape(-1)[idx] - z[f"smean__{key}"]))
                              / max(float(z[f"maxabs_mean__{key}"]), 1e-300))
        vs, vrs = v.reshape(-1)[idx], z[f"svar__{key}"]
        d["var_rel"] = float(np.max(np.abs(vs - vrs)) / max(float(z[f"maxabs_var__{key}"]), 1e-300))
        j = int(np.argmax(np.abs(vs - vrs)))
        d["worst_entry"] = [int(idx[j]), float(vs[j]), float(vrs[j]), float(m.reshape(-1)[idx][j])]
        d["norm_var_rel"] = float(abs(np.linalg.norm(v) - float(z[f"norm_var__{key}"]))
                                  / max(float(z[f"norm_var__{key}"]), 1e-300))
    out["keys"][key] = d
bad = sorted(out["keys"].items(), key=lambda kv: -kv[1]["var_rel"])[:12]
out["worst_var"] = bad
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cfg4_subset.json", "w"), indent=1)
print(json.dumps({k: out[k] for k in ("lambda_rel_max", "iters_mean", "iters_ref_mean", "sum_w")}))
for k, d in bad:
    print(k, d)
