"""Per-system flux-basis block errors vs the golden fixture (debug helper)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

from conftest import case_from_golden, golden  # noqa: E402
from paper_1802_06263_b200.interface import SweepEngine, get_plan  # noqa: E402

name = sys.argv[1]
z = golden(name)
_, problem, grid, _ = case_from_golden(name)
plan = get_plan(problem, grid)
eng = SweepEngine(plan)
eng.kl_fields()
eng.build_bases()
blocks = eng.blocks.cpu().numpy()
for idx, (s, l) in enumerate(eng.systems):
    key = f"B__{s}__{l}"
    if key in z and problem.layout.physics(s) == "stokes":
        nd = int(plan.ndof[s])
        B = blocks[eng.sys_boff[idx]: eng.sys_boff[idx] + nd * nd].reshape(nd, nd).T
        p = plan.patterns[s]
        print(s, "nb", p.nb, "n", p.n, "err %.2e" % (np.max(np.abs(B - z[key])) / np.max(np.abs(z[key]))),
              "asym %.2e" % (np.max(np.abs(B - B.T)) / np.max(np.abs(B))))
