"""cfg4 Method S3 on sampled collocation points (device), optionally checked
against tests/golden/cfg4_points.npz (made by tests/golden/make_cfg4_points.py).

usage: python tools/cfg4_points.py [k ...]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1802_06263_b200.adapter import load_config  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan, hist_padded  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                    "golden", "cfg4_points.npz")


def main():
    z = np.load(GOLD) if os.path.exists(GOLD) else None
    pts = [int(a) for a in sys.argv[1:]] or (list(z["points"]) if z is not None else [0, 1])
    t = time.time()
    problem, grid, _ = load_config("configs/cfg4.json")
    plan = get_plan(problem, grid)
    print(f"setup+plan {time.time() - t:.1f} s, n_lambda {plan.n_lambda}, n_real {grid.n_real}")
    eng = SweepEngine(plan, keep_fields=False)
    torch.cuda.synchronize()
    t = time.time()
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    torch.cuda.synchronize()
    print(f"bases {1e3 * (time.time() - t):.1f} ms")
    nl = plan.n_lambda
    kernels = ["cta", "multi"]
    for kern in kernels:
        for k in pts:
            torch.cuda.synchronize()
            t = time.time()
            lam, iters, status, hist, _ = eng.solve_points(1e-11, max(50, 10 * nl), k0=k,
                                                           n_pts=1, kernel=kern)
            torch.cuda.synchronize()
            dt = time.time() - t
            lam = lam.cpu().numpy()[0]
            it, st = int(iters.cpu().numpy()[0]), int(status.cpu().numpy()[0])
            h = hist_padded(hist, iters).cpu().numpy()[0]
            msg = f"[{kern}] point {k}: {it} iterations, status {st}, {1e3 * dt:.0f} ms"
            if z is not None and k in list(z["points"]):
                j = list(z["points"]).index(k)
                ref = z["lambda"][j]
                head = z["res_head"][j]
                rel = np.abs(h[:len(head)] - head[:min(len(head), it)]) / head[:min(len(head), it)] \
                    if it >= len(head) else np.abs(h[:it] - head[:it]) / head[:it]
                first = int(np.argmax(rel > 1e-6)) if np.any(rel > 1e-6) else len(rel)
                msg += (f", lambda rel err {np.linalg.norm(lam - ref) / np.linalg.norm(ref):.2e}"
                        f" (ref {int(z['iters'][j])} iterations, converged "
                        f"{bool(z['converged'][j])}); residual head agrees to 1e-6 for the "
                        f"first {first} iterations, last residual {h[min(it, h.shape[0]) - 1]:.3e}"
                        f" (ref {float(z['last_residual'][j]):.3e})")
            print(msg, flush=True)


if __name__ == "__main__":
    main()
