"""cfg4 moment goldens on a strided point subset, made by running the REFERENCE.

The full cfg4 Method-S3 sweep (54,273 points, n_lambda = 2,720, 13k-75k CG
iterations per point) is days of CPU, so this runs the reference
(`sdmortar`, imported from /root/reference in the build container) on every
STRIDE-th collocation point: the sub-grid G_P = (points[P], weights[P],
local_indices[.][P]) with the full grid's local tables. `run_method(problem,
G_P, "S3", ...)` on that grid is what this computes, with the work split over
processes:

* bases / operators exactly as `_prepare_s3` builds them (interface.py:349-397),
  but only for the (sid, loc) pairs the subset touches (Stokes frozen at y = 0,
  built once in the parent before the fork);
* per point, in order: `compute_rhs` (166-177), `cg_solve` with
  `basis_apply` (107-139, 238-247) at the config's tol and max_iter,
  `recover_fields` + `_fields_dict` (250-268), and the MomentAccumulator
  update `s += w v; q += w v v` (moments.py:25-38);
* processes take contiguous chunks of the subset and accumulate their chunk
  in point order; chunk sums are added in chunk order. The only difference
  from one sequential accumulator is the association of that last sum, far
  below the reference's own reorder floor (next item);
* the reorder floor: every point solved a second time with the GEMV column
  order inside basis_apply reversed (as make_golden.py does), moments
  accumulated the same way; per key the relative difference of the two
  finalized results is stored (`floor_*`).

Stored (tests/golden/cfg4_moments.npz): the subset, per-point lambda (float64),
iteration counts, first residuals, every key's L2 norm of mean/var, full
mean/var arrays of lambda and of the sids in KEEP_SIDS, and for every other
key a fixed sample of entries.

usage (build container):  OMP_NUM_THREADS=1 python tests/golden/make_cfg4_moments.py [--stride 64] [--procs 7] [--limit N]
"""
import argparse
import collections
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

import sdmortar.interface as ref_iface  # noqa: E402
from sdmortar.collocation import CollocationGrid  # noqa: E402
from sdmortar.config import build_from_config, parse_config  # noqa: E402
from sdmortar.moments import MomentAccumulator  # noqa: E402

KEEP_SIDS = tuple(range(0, 128, 8))
N_SAMPLE = 128
HEAD = 64
DARCY_CACHE = 600

G = {}          # problem, grid, ... shared with the forked workers


def subset_grid(grid, pts):
    """The collocation grid restricted to the points `pts` (same local tables)."""
    return CollocationGrid(grid.kind, grid.points[pts], grid.weights[pts], grid.splits,
                           [li[pts] for li in grid.local_indices], list(grid.local_counts),
                           list(grid.local_points))


def _reversed_basis_apply(space, bases):
    def apply_fn(lam):
        out = np.zeros(space.n_dof)
        for dofs, B in bases:
            out[dofs] += B[:, ::-1] @ lam[dofs][::-1]
        return out
    return apply_fn


def _build(sid, loc):
    problem, grid, stats = G["problem"], G["grid"], G["stats"]
    lay = problem.layout
    zero = np.zeros(grid.n_dims)
    if lay.blocks[sid].physics == "darcy":
        r = lay.blocks[sid].kl_region
        y = zero.copy()
        y[grid.region_slice(r)] = grid.local_points[r][loc]
        c = problem.meshes[sid].centroids
        Kf = {sid: problem.perm.realize(r, c[:, 0], c[:, 1], y)}
    else:
        Kf = G["K0"]
    op = problem.assemble_subdomain(sid, Kf)
    return op, ref_iface.compute_flux_basis(problem, sid, op, stats)


def _get(sid, loc):
    fixed = G["fixed"]
    if (sid, loc) in fixed:
        return fixed[(sid, loc)]
    lru = G.setdefault("lru", collections.OrderedDict())
    if (sid, loc) in lru:
        lru.move_to_end((sid, loc))
        return lru[(sid, loc)]
    v = _build(sid, loc)
    lru[(sid, loc)] = v
    if len(lru) > DARCY_CACHE:
        lru.popitem(last=False)
    return v


def _solve_point(k, apply_maker):
    problem, grid, stats, tol, max_iter = (G["problem"], G["grid"], G["stats"], G["tol"],
                                           G["max_iter"])
    n_sub = problem.layout.n_subdomains
    built = [_get(s, ref_iface._local_of(problem, grid, s, k)) for s in range(n_sub)]
    ops = [b[0] for b in built]
    with ref_iface._Pool(1) as pool:
        bars, g = ref_iface.compute_rhs(problem, ops, pool, stats)
        lam, n_iter, res = ref_iface.cg_solve(apply_maker(problem.space, [b[1] for b in built]),
                                              g, tol=tol, max_iter=max_iter)
        per_sid = ref_iface.recover_fields(problem, ops, bars, lam, pool, stats)
    return lam, n_iter, res, ref_iface._fields_dict(problem, per_sid, lam)


def _acc(sums, w, fields):
    # MomentAccumulator.add arithmetic (moments.py:25-38)
    if not sums:
        for key, v in fields.items():
            sums[key] = [np.zeros_like(np.asarray(v, dtype=float)),
                         np.zeros_like(np.asarray(v, dtype=float))]
    for key, v in fields.items():
        v = np.asarray(v, dtype=float)
        sums[key][0] += w * v
        sums[key][1] += w * v * v


def work(chunk):
    t0 = time.time()
    grid = G["grid"]
    acc, acc2 = {}, {}
    out = {"k": [], "lam": [], "iters": [], "head": [], "last": [], "lam2": [], "iters2": []}
    for k in chunk:
        w = grid.weights[k]
        lam, n_iter, res, fields = _solve_point(k, ref_iface.basis_apply)
        _acc(acc, w, fields)
        lam2, n2, _, fields2 = _solve_point(k, _reversed_basis_apply)
        _acc(acc2, w, fields2)
        out["k"].append(k)
        out["lam"].append(lam)
        out["iters"].append(n_iter)
        h = np.zeros(HEAD)
        h[:min(HEAD, len(res))] = res[:HEAD]
        out["head"].append(h)
        out["last"].append(res[-1] if res else 0.0)
        out["lam2"].append(lam2)
        out["iters2"].append(n2)
    print(f"  chunk {chunk[0]}..{chunk[-1]} ({len(chunk)} points): "
          f"{time.time() - t0:.0f} s, iters {min(out['iters'])}-{max(out['iters'])}", flush=True)
    return out, acc, acc2


def _finalize(sums):
    acc = MomentAccumulator()
    acc._sum = {k: v[0] for k, v in sums.items()}
    acc._sumsq = {k: v[1] for k, v in sums.items()}
    return acc.finalize()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--stride", type=int, default=64)
    ap.add_argument("--procs", type=int, default=7)
    ap.add_argument("--limit", type=int, default=0)
    ap.add_argument("--chunk", type=int, default=8)
    ap.add_argument("--out", default=os.path.join(HERE, "cfg4_moments.npz"))
    args = ap.parse_args()
    t0 = time.time()
    cfg = parse_config(os.path.join(REPO, "configs", "cfg4.json"))
    problem, grid, opts = build_from_config(cfg)
    lay = problem.layout
    n_sub = lay.n_subdomains
    pts = np.arange(0, grid.n_real, args.stride)
    if args.limit:
        pts = pts[:args.limit]
    G.update(problem=problem, grid=grid, stats=ref_iface.SolveStats.new("S3", n_sub),
             tol=opts["tol"], max_iter=opts["max_iter"],
             K0=problem.permeability(np.zeros(grid.n_dims)), fixed={})
    print(f"cfg4: {grid.n_real} points, subset {len(pts)} (stride {args.stride}), "
          f"tol {opts['tol']}, max_iter {opts['max_iter']}; setup {time.time() - t0:.0f} s",
          flush=True)
    # operators shared by (nearly) every point, built once before the fork:
    # Stokes (frozen, loc 0) and each Darcy subdomain's most frequent local realization
    for s in range(n_sub):
        if lay.blocks[s].physics == "darcy":
            li = grid.local_indices[lay.blocks[s].kl_region][pts]
            loc = int(np.bincount(li).argmax())
        else:
            loc = 0
        G["fixed"][(s, loc)] = _build(s, loc)
    print(f"shared operators built: {time.time() - t0:.0f} s", flush=True)
    chunks = [list(pts[i:i + args.chunk]) for i in range(0, len(pts), args.chunk)]
    ctx = mp.get_context("fork")
    with ctx.Pool(args.procs) as pool:
        results = pool.map(work, chunks, chunksize=1)
    acc, acc2 = {}, {}
    rec = {k: [] for k in results[0][0]}
    for out, a, a2 in results:              # chunk order = point order
        for k in rec:
            rec[k] += out[k]
        for dst, src in ((acc, a), (acc2, a2)):
            for key, (s, q) in src.items():
                if key not in dst:
                    dst[key] = [np.zeros_like(s), np.zeros_like(q)]
                dst[key][0] += s
                dst[key][1] += q
    mom, mom2 = _finalize(acc), _finalize(acc2)
    res = {"points": pts, "stride": np.array(args.stride), "n_real_full": np.array(grid.n_real),
           "tol": np.array(opts["tol"]), "max_iter": np.array(opts["max_iter"]),
           "lambda": np.array(rec["lam"]), "iters": np.array(rec["iters"]),
           "res_head": np.array(rec["head"]), "last_residual": np.array(rec["last"]),
           "iters_rev": np.array(rec["iters2"]),
           "weights": grid.weights[pts], "keep_sids": np.array(KEEP_SIDS)}
    lam, lam2 = res["lambda"], np.array(rec["lam2"])
    res["floor_lambda"] = np.array(np.max(np.abs(lam2 - lam)) / np.max(np.abs(lam)))
    rng = np.random.default_rng(2718)
    keys = sorted(mom)
    res["keys"] = np.array(keys)
    for key in keys:
        m, v = mom[key]
        m2, v2 = mom2[key]
        res[f"norm_mean__{key}"] = np.array(np.linalg.norm(m))
        res[f"norm_var__{key}"] = np.array(np.linalg.norm(v))
        res[f"floor_mean__{key}"] = np.array(np.linalg.norm(m2 - m) / max(np.linalg.norm(m), 1e-300))
        res[f"floor_var__{key}"] = np.array(np.linalg.norm(v2 - v) / max(np.linalg.norm(v), 1e-300))
        res[f"floor_meanmax__{key}"] = np.array(np.max(np.abs(m2 - m)) / max(np.max(np.abs(m)), 1e-300))
        res[f"floor_varmax__{key}"] = np.array(np.max(np.abs(v2 - v)) / max(np.max(np.abs(v)), 1e-300))
        sid = None if key == "lambda" else int(key.split(":")[0])
        if sid is None or sid in KEEP_SIDS:
            res[f"mean__{key}"] = m
            res[f"var__{key}"] = v
        else:
            flat = m.reshape(-1)
            idx = np.sort(rng.choice(flat.size, size=min(N_SAMPLE, flat.size), replace=False))
            res[f"idx__{key}"] = idx
            res[f"smean__{key}"] = flat[idx]
            res[f"svar__{key}"] = v.reshape(-1)[idx]
            res[f"maxabs_mean__{key}"] = np.array(np.max(np.abs(m)))
            res[f"maxabs_var__{key}"] = np.array(np.max(np.abs(v)))
    np.savez_compressed(args.out, **res)
    worst = max(float(res[f"floor_mean__{k}"]) for k in keys)
    worstv = max(float(res[f"floor_var__{k}"]) for k in keys)
    print(f"wrote {args.out} ({os.path.getsize(args.out) / 1e6:.2f} MB): iters "
          f"{res['iters'].min()}-{res['iters'].max()} mean {res['iters'].mean():.0f}; "
          f"floor lambda {float(res['floor_lambda']):.2e}, worst key floor mean {worst:.2e} "
          f"var {worstv:.2e}; {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
