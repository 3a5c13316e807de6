"""Mean CG iterations of the device S3 sweep vs the reference's (golden) on
the golden configs (unpreconditioned CG at tol 1e-11: roundoff moves them)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from conftest import case_from_golden
from paper_1802_06263_b200.interface import run_method
for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    z = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
    _, problem, grid, _ = case_from_golden(name)
    res = run_method(problem, grid, method="S3", tol=1e-11)
    it = np.array(res.stats.cg_iters)
    ref = z["s3_iters"]
    keep = z["s3_points"]
    ref = ref[keep] if len(ref) != len(keep) else ref     # (iterations of every point, lambda of the kept ones)
    L = np.array(res.lambdas)[keep]
    print(f"{name}: device mean {it[keep].mean():.1f} vs reference {ref.mean():.1f} "
          f"({100 * (it[keep].mean() / ref.mean() - 1):+.2f}%), per-point diff mean "
          f"{np.mean(it[keep] - ref):+.1f}, lambda rel "
          f"{np.linalg.norm(L - z['s3_lambda']) / np.linalg.norm(z['s3_lambda']):.2e}")
