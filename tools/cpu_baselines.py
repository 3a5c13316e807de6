"""CPU baselines of the reference's S3 algorithm (oracle/s3_cpu.py, 1 thread)
for every BASELINE config, on bounded samples, beside the
device numbers of the same round. Run on the GPU box's host.

* pre-loop: a sample of (sid, loc) systems per physics -- assembly + SuperLU
  factor + one backsolve per mortar dof (compute_flux_basis) -- timed and
  extrapolated to every system of the config;
* main loop: the first points of the grid (bar solves, CG on the bases,
  star-solve recovery, moments) timed and extrapolated to N_real (cfg4's
  hardest points take >3x the mean iterations; the sample is the grid's
  first points, as SURVEY 8d prescribes).

usage: python tools/cpu_baselines.py [--out profiles/r01/cpu_baselines.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402

from oracle import s3_cpu  # noqa: E402
import paper_1802_06263_b200._ref  # noqa: E402,F401  (puts sdmortar on the path)
from sdmortar.collocation import build_tensor_grid  # noqa: E402
from paper_1802_06263_b200.adapter import load_config  # noqa: E402

PLAN = {  # config: (systems sampled per physics, points sampled)
    "cfg1": (None, None), "cfg2": (None, None), "cfg3": (6, 8), "cfg4": (3, 2),
    "cfg5": (8, 0)}


def sample_systems(problem, grid, per_phys, local_pts=None):
    """Time (assemble + flux basis) on a sample of systems per physics;
    return (seconds per system by physics, count of systems by physics,
    local solves per system by physics)."""
    plan = s3_cpu.s3_plan(problem, grid)
    if local_pts is not None:                  # cfg5: 729 tensor points per region
        zero = np.zeros(grid.n_dims)
        plan = {}
        for sid in range(problem.layout.n_subdomains):
            r = problem.layout.blocks[sid].kl_region
            pts = []
            for loc in local_pts:
                y = zero.copy()
                y[grid.region_slice(r)] = loc
                pts.append(y)
            plan[sid] = pts
    K0 = s3_cpu.mean_field_K(problem, grid.n_dims)
    by = {}
    for sid, pts in plan.items():
        ph = problem.layout.blocks[sid].physics
        by.setdefault(ph, []).extend((sid, y) for y in pts)
    sec, cnt, solves = {}, {}, {}
    for ph, items in by.items():
        cnt[ph] = len(items)
        take = items if per_phys is None else [items[i] for i in
                                                np.linspace(0, len(items) - 1,
                                                            min(per_phys, len(items)),
                                                            dtype=int)]
        t0 = time.perf_counter()
        nd = 0
        for sid, y in take:
            Kf = {sid: s3_cpu.realize(problem, sid, y)} if sid in K0 else K0
            op = s3_cpu.assemble(problem, sid, Kf)
            dofs, B = s3_cpu.flux_basis(problem, sid, op)
            nd += B.shape[0]
        sec[ph] = (time.perf_counter() - t0) / len(take)
        solves[ph] = nd / len(take)
    return sec, cnt, solves


def time_points(problem, grid, pts):
    """The S3 main loop (interface.py:306-341) on `pts`: the systems the points
    use are built first (untimed; the pre-loop estimate covers them), then
    rhs, CG, recovery and moments are timed per point."""
    n_sub = problem.layout.n_subdomains
    K0 = s3_cpu.mean_field_K(problem, grid.n_dims)
    zero = np.zeros(grid.n_dims)
    cache = {}

    def build(sid, loc):
        if (sid, loc) not in cache:
            if sid in K0:
                r = problem.layout.blocks[sid].kl_region
                y = zero.copy()
                y[grid.region_slice(r)] = grid.local_points[r][loc]
                Kf = {sid: s3_cpu.realize(problem, sid, y)}
            else:
                Kf = K0
            op = s3_cpu.assemble(problem, sid, Kf)
            cache[(sid, loc)] = (op, s3_cpu.flux_basis(problem, sid, op))
        return cache[(sid, loc)]

    def pick(k):
        built = [build(s, s3_cpu.local_of(problem, grid, s, k)) for s in range(n_sub)]
        return [b[0] for b in built], [b[1] for b in built]

    for k in pts:
        pick(k)
    t0 = time.perf_counter()
    r = s3_cpu._sweep(problem, grid, pick, 1e-11, max(50, 10 * problem.space.n_dof) * 8,
                      pts, False)
    return (time.perf_counter() - t0) / len(pts), [int(x) for x in r["iters"]]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "cpu_baselines.json"))
    ap.add_argument("--configs", nargs="*", default=list(PLAN))
    a = ap.parse_args()
    out = {"cores": 1, "threads": "1 BLAS thread (threadpoolctl)", "kind": "port",
           "note": "oracle/s3_cpu.py restates sdmortar's S3 (SuperLU, numpy CG); bounded "
                   "samples extrapolated linearly (SURVEY 8d)", "configs": {}}
    for cfg in a.configs:
        per_phys, n_pts = PLAN[cfg]
        problem, grid, _ = load_config(os.path.join(ROOT, "configs", f"{cfg}.json"))
        local = build_tensor_grid([3] * 6).points if cfg == "cfg5" else None
        with threadpool_limits(limits=1):
            sec, cnt, solves = sample_systems(problem, grid, per_phys, local)
            pre = sum(sec[p] * cnt[p] for p in sec)
            res = {"systems": cnt, "s_per_system": sec,
                   "pre_loop_s_est": pre,
                   "local_solves_per_s": sum(solves[p] * cnt[p] for p in sec) / pre,
                   "sampled_systems_per_physics": per_phys or "all"}
            if cfg != "cfg5":
                pts = list(range(grid.n_real)) if n_pts is None else list(range(n_pts))
                per_point, iters = time_points(problem, grid, pts)
                res.update(points_timed=len(pts), cg_iters=iters,
                           main_loop_s_per_point=per_point,
                           sweep_s_est=pre + per_point * grid.n_real,
                           realizations_per_s=grid.n_real / (pre + per_point * grid.n_real))
        out["configs"][cfg] = res
        print(cfg, json.dumps(res), flush=True)
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
