import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
from paper_1802_06263_b200.adapter import load_config
from paper_1802_06263_b200.interface import run_method
problem, grid, _ = load_config("configs/cfg2.json")
for _ in range(3): run_method(problem, grid, method="S3", tol=1e-11)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): run_method(problem, grid, method="S3", tol=1e-11)
print("per call ms", (time.perf_counter()-t)/10*1e3)
pr=cProfile.Profile(); pr.enable()
for _ in range(10): run_method(problem, grid, method="S3", tol=1e-11)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
