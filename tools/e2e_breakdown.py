"""Where run_method's end-to-end time goes (cfg2 S3): host time before the
first launch, the launch phase, the wait, and the host work after the wait.
python tools/e2e_breakdown.py"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1802_06263_b200.interface as itf  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402

acc = collections.defaultdict(float)
marks = {}


def wrap(cls, name):
    f = getattr(cls, name)

    def g(*a, **k):
        t = time.perf_counter()
        marks.setdefault(name, t)
        r = f(*a, **k)
        acc[name] += time.perf_counter() - t
        return r
    setattr(cls, name, g)


for n in ("kl_fields", "build_bases", "solve_points", "moments_launch", "check_info",
          "moments_finish"):
    wrap(itf.SweepEngine, n)
wrap(itf._SweepStatic, "refresh_inputs")
problem, grid, _ = load_config(os.path.join("configs", "cfg2.json"))
for _ in range(5):
    itf.run_method(problem, grid, method="S3", tol=1e-11)
torch.cuda.synchronize()
acc.clear()
N = 20
tot = 0.0
first = 0.0
for _ in range(N):
    marks.clear()
    t0 = time.perf_counter()
    itf.run_method(problem, grid, method="S3", tol=1e-11)
    t1 = time.perf_counter()
    tot += t1 - t0
    first += marks["kl_fields"] - t0
print(f"run_method {tot / N * 1e3:.3f} ms per call; start -> first launch "
      f"{first / N * 1e3:.3f} ms")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
    print(f"  {k:16s} {v / N * 1e3:.3f} ms")
