"""Generate the golden fixtures by running the REFERENCE package (sdmortar).

Run once in the build container, where the read-only reference is mounted:

    PYTHONPATH=/root/reference/pkg/src OMP_NUM_THREADS=1 \
        python tests/golden/make_golden.py [case ...]

Nothing at test time imports the reference: the fixtures below are what
travels. Each `<case>.npz` holds, for one configuration:

* setup pins: collocation points/weights/local tables, mortar dof maps
  (`sub_dofs`), interface list -- checked bit-exact against our host setup;
* per-(sid, loc) K fields and flux-basis blocks `B` from
  `compute_flux_basis` (reference interface.py:218-235);
* a full Method-S3 sweep (`run_method`, interface.py:288-346) at tol 1e-11:
  per-point rhs g, lambda, iteration count, residual history, the moments of
  every field key, and the SolveStats counters;
* the reference's own noise floor: the same sweep with the GEMV column order
  inside `basis_apply` reversed; per-key drift of mean/var is stored so that
  parity tests can judge our device results against it.

Configs are the repo's `configs/cfg*.json`, plus the reference's shipped
`case1_mini`, `darcy_twoblock` configs (read from the mount at generation
time; their parsed, normalised form is stored in the fixture).
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_CONFIGS = "/root/reference/pkg/configs"

import sdmortar.interface as ref_iface  # noqa: E402
from sdmortar.collocation import build_tensor_grid  # noqa: E402
from sdmortar.config import build_from_config, parse_config  # noqa: E402
from sdmortar.interface import SolveStats, compute_flux_basis, run_method  # noqa: E402


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _setup_pins(problem, grid, out, full_grid=True):
    lay = problem.layout
    out["n_lambda"] = np.array(problem.space.n_dof)
    out["n_real"] = np.array(grid.n_real)
    out["local_counts"] = np.array(grid.local_counts)
    out["ifaces"] = np.array([[g.index, g.i, g.j, "sd dd ss".split().index(g.kind),
                               0 if g.axis == "x" else 1, g.normal_sign]
                              for g in lay.interfaces])
    dofs = [problem.space.sub_dofs(lay, s) for s in range(lay.n_subdomains)]
    out["sub_dofs"] = np.concatenate(dofs)
    out["sub_dofs_ptr"] = np.cumsum([0] + [len(d) for d in dofs])
    out["sha_points"] = np.array(_sha(grid.points))
    out["sha_weights"] = np.array(_sha(grid.weights))
    out["sha_local"] = np.array(_sha(np.stack(grid.local_indices)))
    if full_grid:
        out["grid_points"] = grid.points
        out["grid_weights"] = grid.weights
        out["grid_local"] = np.stack(grid.local_indices)


def _plan_points(problem, grid, sid):
    """Stochastic points S3 plans for one subdomain (interface.py:360-373)."""
    zero = np.zeros(grid.n_dims)
    block = problem.layout.blocks[sid]
    if block.physics != "darcy":
        return [zero]
    pts = []
    for loc in grid.local_points[block.kl_region]:
        y = zero.copy()
        y[grid.region_slice(block.kl_region)] = loc
        pts.append(y)
    return pts


def _block(problem, grid, sid, y):
    lay = problem.layout
    if lay.blocks[sid].physics == "darcy":
        c = problem.meshes[sid].centroids
        K = problem.perm.realize(lay.blocks[sid].kl_region, c[:, 0], c[:, 1], y)
        Kf = {sid: K}
    else:
        K = None
        Kf = problem.permeability(np.zeros(grid.n_dims))
    op = problem.assemble_subdomain(sid, Kf)
    stats = SolveStats.new("S3", lay.n_subdomains)
    _, B = compute_flux_basis(problem, sid, op, stats)
    return K, B


def _blocks(problem, grid, out, select=None):
    for sid in range(problem.layout.n_subdomains):
        pts = _plan_points(problem, grid, sid)
        locs = range(len(pts)) if select is None else select(sid, len(pts))
        for loc in locs:
            K, B = _block(problem, grid, sid, pts[loc])
            out[f"B__{sid}__{loc}"] = B
            if K is not None:
                out[f"K__{sid}__{loc}"] = K


class _Recorder:
    """Wrap cg_solve to capture the per-point right-hand side."""

    def __init__(self):
        self.g = []
        self.orig = ref_iface.cg_solve

    def __call__(self, apply_fn, g, tol=1e-9, max_iter=None):
        self.g.append(np.array(g))
        return self.orig(apply_fn, g, tol=tol, max_iter=max_iter)


def _reversed_basis_apply(space, bases):
    def apply_fn(lam):
        out = np.zeros(space.n_dof)
        for dofs, B in bases:
            out[dofs] += B[:, ::-1] @ lam[dofs][::-1]
        return out
    return apply_fn


def _sweep(problem, grid, tol, out, floor=True, keep_points=None):
    rec = _Recorder()
    ref_iface.cg_solve = rec
    t0 = time.perf_counter()
    try:
        res = run_method(problem, grid, method="S3", tol=tol)
    finally:
        ref_iface.cg_solve = rec.orig
    out["s3_wall"] = np.array(time.perf_counter() - t0)
    lam = np.array(res.lambdas)
    keep = np.arange(grid.n_real) if keep_points is None else keep_points
    out["s3_points"] = keep
    out["s3_lambda"] = lam[keep]
    out["s3_g"] = np.array(rec.g)[keep]
    out["s3_iters"] = np.array(res.stats.cg_iters)
    hist = [np.array(r) for r in res.residuals]
    out["s3_res_ptr"] = np.cumsum([0] + [len(h) for h in hist])
    out["s3_res"] = np.concatenate(hist) if hist else np.zeros(0)
    for k, (m, v) in res.moments.items():
        out[f"mean__{k}"] = m
        out[f"var__{k}"] = v
    out["stats_backsolves"] = res.stats.backsolves
    out["stats_factorizations"] = res.stats.factorizations
    out["stats_basis_backsolves"] = res.stats.basis_backsolves
    if not floor:
        return res
    orig = ref_iface.basis_apply
    ref_iface.basis_apply = _reversed_basis_apply
    try:
        res2 = run_method(problem, grid, method="S3", tol=tol)
    finally:
        ref_iface.basis_apply = orig
    lam2 = np.array(res2.lambdas)
    out["floor_lambda"] = np.array(np.max(np.abs(lam2 - lam)) / np.max(np.abs(lam)))
    for k, (m, v) in res.moments.items():
        m2, v2 = res2.moments[k]
        out[f"floor_mean__{k}"] = np.array(
            np.linalg.norm(m2 - m) / max(np.linalg.norm(m), 1e-300))
        out[f"floor_var__{k}"] = np.array(
            np.linalg.norm(v2 - v) / max(np.linalg.norm(v), 1e-300))
        out[f"floor_varm2__{k}"] = np.array(
            np.max(np.abs(v2 - v)) / max(np.max(m * m), 1e-300))
    out["floor_iters_changed"] = np.array(
        int(np.sum(np.array(res2.stats.cg_iters) != np.array(res.stats.cg_iters))))
    return res


def _load(name):
    path = (os.path.join(REPO, "configs", name + ".json")
            if name.startswith("cfg") else os.path.join(REF_CONFIGS, name + ".json"))
    cfg = parse_config(path)
    return cfg, build_from_config(cfg)


def case(name):
    out = {}
    t0 = time.time()
    cfg, (problem, grid, opts) = _load(name)
    out["config_json"] = np.array(json.dumps(cfg, sort_keys=True))
    tol = 1e-11
    if name in ("cfg1", "cfg2", "case1_mini", "darcy_twoblock"):
        _setup_pins(problem, grid, out)
        _blocks(problem, grid, out)
        _sweep(problem, grid, tol, out)
    elif name == "cfg3":
        _setup_pins(problem, grid, out)
        _blocks(problem, grid, out,
                select=lambda sid, n: [0, n // 2, n - 1] if n > 1 else [0])
        res = _sweep(problem, grid, tol, out, keep_points=np.arange(0, grid.n_real, 8))
        # moments: keep lambda and a sample of subdomains to stay small
        keepk = {"lambda"} | {f"{s}:{f}" for s in (0, 9, 16, 17, 31)
                             for f in ("u", "p", "cv", "cp")}
        for k in list(out):
            for pre in ("mean__", "var__", "floor_mean__", "floor_var__", "floor_varm2__"):
                if k.startswith(pre) and k[len(pre):] not in keepk:
                    del out[k]
    elif name == "cfg4":
        _setup_pins(problem, grid, out, full_grid=False)
        out["grid_weights_head"] = grid.weights[:4096]
        out["grid_local_head"] = np.stack(grid.local_indices)[:, :4096]
        sel = {64: [0, 1, 100, 288], 127: [0, 5], 0: [0], 21: [0]}
        _blocks(problem, grid, out, select=lambda sid, n: sel.get(sid, []))
    elif name == "cfg5":
        _setup_pins(problem, grid, out)
        # basis-only: local points = build_tensor_grid([3]*6) per region
        loc_grid = build_tensor_grid([3] * 6)
        out["loc_points"] = loc_grid.points
        lay = problem.layout
        for sid in range(lay.n_subdomains):
            for loc in (0, 1, 364, 728):
                y = np.zeros(problem.perm.n_dims)
                y[problem.perm.region_slice(lay.blocks[sid].kl_region)] = loc_grid.points[loc]
                K, B = _block(problem, grid, sid, y)
                out[f"B__{sid}__{loc}"] = B
                if sid == 0:
                    out[f"K__{sid}__{loc}"] = K
    else:
        raise SystemExit(f"unknown case {name}")
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print(f"{name}: {len(out)} arrays, {os.path.getsize(path) / 1e6:.2f} MB, "
          f"{time.time() - t0:.1f} s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg1", "darcy_twoblock", "case1_mini", "cfg2", "cfg5",
                             "cfg4", "cfg3"]
    for n in names:
        case(n)
