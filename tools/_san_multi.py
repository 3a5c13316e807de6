import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.getcwd() + "/tests")
import numpy as np, torch
from conftest import case_from_golden
from paper_1802_06263_b200.interface import S3Engine, get_plan
_, problem, grid, _ = case_from_golden(sys.argv[1])
plan = get_plan(problem, grid)
eng = S3Engine(plan); eng.kl_fields(); eng.build_bases(); eng.check_info()
lam, it, st, h, g = eng.solve_points(1e-11, 500, keep_g=True, kernel="multi")
torch.cuda.synchronize()
print("status", np.bincount(st.cpu().numpy()), "iters", it.cpu().numpy()[:8])
