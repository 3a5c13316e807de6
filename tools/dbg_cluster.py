import os, sys
ROOT='/root/repo'; sys.path.insert(0, ROOT); sys.path.insert(0, ROOT+'/tests')
import numpy as np, torch
from conftest import case_from_golden
from paper_1802_06263_b200.interface import SweepEngine, get_plan
shp = tuple(int(v) for v in sys.argv[1].split('x'))
name = sys.argv[2] if len(sys.argv) > 2 else 'cfg1'
_, problem, grid, _ = case_from_golden(name)
plan = get_plan(problem, grid)
eng = SweepEngine(plan, keep_fields=False)
eng.kl_fields(); eng.build_bases(); eng.check_info()
from paper_1802_06263_b200 import _lib
_lib.load().mfb_debug_cluster(int(os.environ.get('DBG','0')))
lam, it, st, hist, g = eng.solve_points(1e-11, 2000, kernel="cluster", cluster_shape=[shp], n_pts=int(sys.argv[3]) if len(sys.argv)>3 else None)
torch.cuda.synchronize()
print(shp, name, it.cpu().numpy()[:10], st.cpu().numpy()[:10])
