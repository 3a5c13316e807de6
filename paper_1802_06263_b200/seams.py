"""The reference's secondary seams, on the device.

`run_method` is the primary seam. These are the other public entry points of
`sdmortar.interface` a caller may hold, with the reference's signatures,
return types and errors:

* `solve_realization(problem, y, tol, max_iter, workers)` (interface.py:417-
  437, exported as `sdmortar.solve_realization`): one deterministic
  realization. On the device it is a one-point Method-S2 sweep -- every
  subdomain's system at y, its flux basis, the interface CG, the recovered
  fields -- whose moments with weight 1 are the fields themselves. The
  reference solves the same interface problem matrix-free (S1); the answers
  agree to the CG tolerance (S1 = S2 = S3, test_acceptance.py:124-141).
* `basis_apply(space, bases)` (238-247): S p from per-subdomain (dofs, B)
  blocks. Returns a device operator (blocks uploaded once) that is also a
  plain callable `apply_fn(lam) -> S lam` (mfb_basis_apply).
* `cg_solve(apply_fn, g, tol, max_iter)` (107-139): with a device operator
  from `basis_apply` the CG runs on the device (mfb_cg_batched, one point,
  the reference's stopping/breakdown/zero-rhs rules and ConvergenceError
  carrying the residual history). Any other Python callable is the
  reference's own host function, unchanged: it has no device form.
* `compute_flux_basis(problem, sid, op, stats)` (218-235): with a device
  operator from `assemble_subdomain(problem, sid, K_fields)` (the
  reference's problem.assemble_subdomain signature) the block comes from the
  device system solve of that subdomain with exactly those K fields; a
  reference operator goes to the reference's function.
"""

import numpy as np

from . import _lib
from ._ref import sdmortar
from .errors import ConvergenceError
from .plan import _dev, _ptr

_ri = sdmortar.interface


def _one_point_grid(problem, y):
    """A CollocationGrid holding the single point y (weight 1)."""
    from sdmortar.collocation import CollocationGrid
    splits = tuple(int(r.n_term) for r in problem.perm.regions)
    y = np.asarray(y, dtype=np.float64).reshape(1, -1)
    loc_idx, loc_cnt, loc_pts, lo = [], [], [], 0
    for n_i in splits:
        loc_idx.append(np.zeros(1, dtype=int))
        loc_cnt.append(1)
        loc_pts.append(y[:, lo:lo + n_i].copy())
        lo += n_i
    return CollocationGrid("tensor", y, np.array([1.0]), splits, loc_idx, loc_cnt, loc_pts)


def _fields(moments, n_sub):
    per_sid = []
    for s in range(n_sub):
        per_sid.append({name: np.array(moments[k][0]) for k in moments
                        if k.startswith(f"{s}:") for name in [k.split(":")[1]]})
    return per_sid


def solve_realization(problem, y=None, tol=1e-9, max_iter=None, workers=1):
    """One deterministic realization (reference interface.py:417-437): returns
    (per-subdomain field dicts u, p, cv, cp; lambda; SolveStats in the
    reference's S1 counting)."""
    from .interface import SolveStats, run_method
    n_sub = problem.layout.n_subdomains
    if y is None:
        y = np.zeros(problem.perm.n_dims)
    grid = _one_point_grid(problem, y)
    res = run_method(problem, grid, method="S2", tol=tol, max_iter=max_iter, workers=workers)
    n_iter = int(res.stats.cg_iters[0])
    stats = SolveStats.new("S1", n_sub)
    stats.n_real = 1
    stats.cg_iters = [n_iter]
    # the reference: one factorization per subdomain, the bar solve, one star
    # solve per CG iteration (direct_apply) and the recovery
    stats.factorizations[:] = 1
    stats.backsolves[:] = n_iter + 2
    stats.wall_seconds[:] = res.stats.wall_seconds
    return _fields(res.moments, n_sub), np.array(res.lambdas[0]), stats


class DeviceBasisOperator:
    """S from stored per-subdomain blocks, resident on the device (the
    reference's basis_apply closure, interface.py:238-247)."""

    def __init__(self, space, bases):
        import torch

        from .interface import cg_tasks
        self.space = space
        self.n = int(space.n_dof)
        dofs = [np.asarray(d, dtype=np.int64) for d, _ in bases]
        nd = np.array([len(d) for d in dofs], dtype=np.int64)
        self.n_sub = len(dofs)
        self.ndof = nd
        self.dof_ptr = np.concatenate([[0], np.cumsum(nd)]).astype(np.int32)
        self.dof_map = np.concatenate(dofs).astype(np.int32) if dofs else np.zeros(0, np.int32)
        _, sides, _, _ = cg_tasks(self.n_sub, nd, self.dof_ptr, self.dof_map, self.n)
        self.sides = sides
        blk = np.concatenate([[0], np.cumsum(nd * nd)]).astype(np.int64)
        pool = np.concatenate([np.ascontiguousarray(np.asarray(B, dtype=np.float64).T).ravel()
                               for _, B in bases]) if bases else np.zeros(0)
        i32, i64, f64 = torch.int32, torch.int64, torch.float64
        self.d = {"ndof": _dev(nd.astype(np.int32), i32), "dof_ptr": _dev(self.dof_ptr, i32),
                  "dof_map": _dev(self.dof_map, i32), "sides": _dev(sides.ravel(), i32),
                  "blk": _dev(blk[:-1], i64), "blocks": _dev(pool, f64),
                  "region": _dev(-np.ones(self.n_sub, dtype=np.int32), i32),
                  "h_base": _dev(self.dof_ptr[:-1].astype(np.int64), i64),
                  "local": _dev(np.zeros((1, 1), dtype=np.int32), i32)}
        self.n_rows = int(self.dof_ptr[-1])

    def __call__(self, lam):
        import torch
        L = _lib.lib()
        p = torch.as_tensor(np.asarray(lam, dtype=np.float64)).to("cuda")
        rows = torch.empty(max(self.n_rows, 1), dtype=torch.float64, device="cuda")
        out = torch.empty(self.n, dtype=torch.float64, device="cuda")
        d = self.d
        _lib.check(L.mfb_basis_apply(self.n, self.n_sub, _ptr(d["ndof"]), _ptr(d["dof_ptr"]),
                                     _ptr(d["dof_map"]), _ptr(d["sides"]), _ptr(d["blk"]),
                                     _ptr(d["blocks"]), _ptr(p), _ptr(rows), _ptr(out), None),
                   "mfb_basis_apply")
        return out.cpu().numpy()

    def cg(self, g, tol, max_iter):
        """The batched CG kernel on the single right-hand side g: g enters as
        the bar jump of the lower side of each dof (the upper side's is 0, so
        the kernel's g = h_lower + h_upper is g exactly)."""
        import torch
        L = _lib.lib()
        g = np.asarray(g, dtype=np.float64)
        hbar = np.zeros(self.n_rows)
        first = self.sides[:, 0]
        rows = self.dof_ptr[first] + self.sides[:, 1]
        hbar[rows] = g
        d = self.d
        d_h = _dev(hbar, torch.float64)
        lam = torch.empty((1, self.n), dtype=torch.float64, device="cuda")
        iters = torch.empty(1, dtype=torch.int32, device="cuda")
        status = torch.empty(1, dtype=torch.int32, device="cuda")
        hist = torch.empty((1, max(max_iter, 1)), dtype=torch.float64, device="cuda")
        nd2 = int(np.sum(self.ndof.astype(np.int64) ** 2))
        reg_nd = int(self.ndof.max()) if self.n_sub and not np.any(self.ndof % 4) else 0
        _lib.check(L.mfb_cg_batched(
            self.n, self.n_sub, _ptr(d["ndof"]), _ptr(d["dof_ptr"]), _ptr(d["dof_map"]),
            _ptr(d["region"]), _ptr(d["blk"]), _ptr(d["h_base"]), _ptr(d["local"]), 1,
            _ptr(d["blocks"]), _ptr(d_h), 0, 1, float(tol), int(max_iter), _ptr(lam),
            _ptr(iters), _ptr(status), _ptr(hist), max(max_iter, 1), None, nd2, reg_nd, None),
            "mfb_cg_batched")
        it, st = int(iters.cpu()[0]), int(status.cpu()[0])
        res = hist.cpu().numpy()[0, :it].tolist()
        return lam.cpu().numpy()[0], it, st, res


def basis_apply(space, bases):
    """S application from stored per-subdomain response matrices (reference
    interface.py:238-247), on the device."""
    return DeviceBasisOperator(space, bases)


def cg_solve(apply_fn, g, tol=1e-9, max_iter=None):
    """Plain CG from x0 = 0 (reference interface.py:107-139): (x, n_iter,
    relative residuals). A device operator (basis_apply) runs on the device;
    any other callable is the reference's host function."""
    if not isinstance(apply_fn, DeviceBasisOperator):
        return _ri.cg_solve(apply_fn, g, tol=tol, max_iter=max_iter)
    n = len(g)
    if max_iter is None:
        max_iter = max(50, 10 * n)
    x, it, st, res = apply_fn.cg(g, tol, max_iter)
    if st == 3:                                  # zero rhs: interface.py:111-113
        return np.zeros(n), 0, []
    if st == 1:
        raise ConvergenceError(f"interface operator is not positive definite "
                               f"(p.Sp <= 0 at iteration {it})", res[:it - 1])
    if st == 2:
        raise ConvergenceError(f"CG did not reach tol {tol:g} in {max_iter} iterations "
                               f"(last residual {res[-1]:.3e})", res)
    return x, it, res


class DeviceSubdomainOperator:
    """A subdomain operator on the device: (problem, sid, K fields) as
    problem.assemble_subdomain takes them (problem.py:98-115); the system is
    built and solved by the sweep kernels when its flux basis is asked for."""

    def __init__(self, problem, sid, K_fields):
        self.problem, self.sid = problem, sid
        self.K_fields = {int(k): np.asarray(v, dtype=np.float64) for k, v in K_fields.items()}
        self.factorizations, self.backsolves = 1, 0


def assemble_subdomain(problem, sid, K_fields):
    """Device counterpart of problem.assemble_subdomain(sid, K_fields)."""
    return DeviceSubdomainOperator(problem, sid, K_fields)


def compute_flux_basis(problem, sid, op, stats):
    """(dofs, B) of subdomain sid (reference interface.py:218-235): with a
    DeviceSubdomainOperator the block is the device system solve of that
    subdomain at its K fields (a one-point S2 sweep state whose K buffer
    takes the given fields before the solve); a reference operator goes to
    the reference's function."""
    if not isinstance(op, DeviceSubdomainOperator):
        return _ri.compute_flux_basis(problem, sid, op, stats)
    import torch

    from .interface import SweepEngine, get_plan
    lay = problem.layout
    grid = _one_point_grid(problem, np.zeros(problem.perm.n_dims))
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, method="S2", keep_fields=False)
    eng.kl_fields()
    st = eng.st
    # the S2 K buffer: row 0 = K0 (k0_len cells), row 1 = realization 0; every
    # Darcy subdomain's cells at k0_off[s] within a row
    K = st.K
    for s in plan.darcy:
        if s in op.K_fields:
            v = torch.as_tensor(op.K_fields[s], device="cuda")
            o = plan.k0_len + plan.k0_off[s]
            K[o:o + v.numel()] = v
    eng.build_bases(sids=[sid])
    eng.check_info()
    nd = int(plan.ndof[sid])
    b0 = int(st.blk_base[sid])
    B = st.blocks[b0:b0 + nd * nd].reshape(nd, nd).T.cpu().numpy()   # stored column-major
    dofs = problem.space.sub_dofs(lay, sid)
    stats.basis_backsolves[sid] += nd
    op.backsolves += nd
    torch.cuda.synchronize()
    return dofs, np.array(B)
