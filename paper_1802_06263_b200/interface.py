"""Drop-in `run_method` for Method S3 on one B200.

Same signature, return type and error behaviour as the reference's
`sdmortar.interface.run_method` (interface.py:288-346): a `RunResult` with
`moments` {key: (mean, var)} over the keys "lambda" and "{sid}:{u,p,cv,cp}",
per-subdomain `SolveStats`, the per-point mortar solutions `lambdas` and CG
residual histories `residuals`. Underneath, every piece of compute runs on
the device through the C ABI (include/mfb.h):

  1. KL kernel: K for every local realization of every region (+ mean field)
  2. one batched launch assembles, factors and solves every (subdomain,
     local realization) system against all mortar columns and the bar rhs,
     then extracts the flux-basis blocks, bar jumps and field responses
  3. one batched CG launch solves all collocation points concurrently
  4. moment kernels (lambda streamed in realization order; fields through
     per-group shifted statistics)

Methods S1 and S2 are not part of this tier's hot path and
raise NotImplementedError -- there is no CPU fallback.
"""

import ctypes
import logging
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConvergenceError, SingularOperatorError, SizeCapError
from .plan import DevicePlan, _dev, _ptr

log = logging.getLogger(__name__)

METHODS = ("S1", "S2", "S3")
_PLAN_CACHE = {}
WORK_BUDGET_BYTES = 8 << 30


@dataclass
class SolveStats:
    """Per-subdomain counters in the reference's semantics (interface.py:35-77).

    Backsolve counts are the reference's S3 identities (interface.py:14-16):
    N_dof_i N_loc(i) basis solves + 2 N_real (bar + recovery), one
    factorization per local realization; the device realises the same
    solves as batched multi-RHS eliminations.
    """

    method: str
    n_sub: int
    factorizations: np.ndarray
    backsolves: np.ndarray
    basis_backsolves: np.ndarray
    cg_iters: list = field(default_factory=list)
    wall_seconds: np.ndarray = None
    n_real: int = 0

    @classmethod
    def new(cls, method, n_sub):
        z = lambda: np.zeros(n_sub, dtype=int)
        return cls(method, n_sub, z(), z(), z(), wall_seconds=np.zeros(n_sub))

    @property
    def cg_iters_total(self):
        return int(sum(self.cg_iters))

    def rows(self):
        return [{"method": self.method, "subdomain": sid,
                 "factorizations": int(self.factorizations[sid]),
                 "backsolves": int(self.backsolves[sid]),
                 "basis_backsolves": int(self.basis_backsolves[sid]),
                 "cg_iters_total": self.cg_iters_total, "n_real": self.n_real,
                 "wall_seconds": float(self.wall_seconds[sid])}
                for sid in range(self.n_sub)]


@dataclass
class RunResult:
    moments: dict
    stats: SolveStats
    lambdas: list
    residuals: list
    grid: object
    timings: dict = field(default_factory=dict)


def _check_basis_cap(sizes_bytes, cap_mb):
    total = sum(sizes_bytes)
    if cap_mb is not None and total > cap_mb * 2 ** 20:
        raise SizeCapError(f"flux basis storage {total / 2 ** 20:.3g} MiB exceeds the "
                           f"cap of {cap_mb:.3g} MiB; raise basis_cap_mb or use method S1")


def get_plan(problem, grid):
    key = (id(problem), id(grid))
    plan = _PLAN_CACHE.get(key)
    if plan is None or plan.problem is not problem or plan.grid is not grid:
        plan = DevicePlan(problem, grid)
        _PLAN_CACHE.clear()
        _PLAN_CACHE[key] = plan
    return plan


class S3Engine:
    """Device state of one S3 sweep; methods map 1:1 onto the C ABI calls."""

    def __init__(self, plan, stream=None):
        import torch
        self.torch = torch
        self.plan = plan
        self.L = _lib.lib()
        self.stream = torch.cuda.current_stream() if stream is None else stream
        self.sp = ctypes.c_void_p(self.stream.cuda_stream)
        self.launches = 0            # kernels launched through the C ABI
        self.timing = False          # record CUDA events around the basis solves
        self.solve_events = []
        self.solve_flops = []

    def _ev(self):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        return ev

    # ------------------------------------------------------------ (1) KL --
    def kl_fields(self):
        """K for every (Darcy sid, loc) system plus the mean-field K0 buffer."""
        torch, plan = self.torch, self.plan
        pb = plan.problem
        lay = pb.layout
        systems = plan.s3_systems()
        koff = np.zeros(len(systems), dtype=np.int64)
        sys_of = {}
        cur = plan.k0_len
        for idx, (s, l) in enumerate(systems):
            sys_of[(s, l)] = idx
            if lay.physics(s) == "darcy":
                koff[idx] = cur
                cur += pb.meshes[s].n_cells
            else:
                koff[idx] = 0                       # Stokes: the K0 buffer
        K = torch.empty(max(cur, 1), dtype=torch.float64, device="cuda")
        self._kl_tabs = []
        for s in plan.darcy:
            r = lay.blocks[s].kl_region
            c = pb.meshes[s].centroids
            phi, mean = pb.perm.mode_table(r, c[:, 0], c[:, 1])
            nt = phi.shape[1]
            xi = np.zeros((1 + int(plan.n_loc[s]), nt))
            xi[1:] = plan.grid.local_points[r][:, :nt]
            d_phi, d_mean, d_xi = (_dev(phi, torch.float64), _dev(mean, torch.float64),
                                   _dev(xi, torch.float64))
            self._kl_tabs.append((d_phi, d_mean, d_xi))
            nc = len(mean)
            # mean field -> K0 slot, local realizations -> their system slots
            self.launches += 2
            _lib.check(self.L.mfb_kl_realize(_ptr(d_phi), _ptr(d_mean), nc, nt, _ptr(d_xi),
                                             1, ctypes.c_void_p(K.data_ptr() + 8 * plan.k0_off[s]),
                                             self.sp), "mfb_kl_realize")
            first = koff[sys_of[(s, 0)]]
            _lib.check(self.L.mfb_kl_realize(
                _ptr(d_phi), _ptr(d_mean), nc, nt,
                ctypes.c_void_p(d_xi.data_ptr() + 8 * nt), int(plan.n_loc[s]),
                ctypes.c_void_p(K.data_ptr() + 8 * int(first)), self.sp), "mfb_kl_realize")
        self.K, self.koff, self.systems = K, koff, systems
        return K

    # ------------------------------------------------------- (2) bases ----
    def build_bases(self, threads=None, keep_fields=True):
        torch, plan = self.torch, self.plan
        systems = self.systems
        pats = plan.patterns
        nsys = len(systems)
        sys_pat = np.array([s for s, _ in systems], dtype=np.int32)
        nd = plan.ndof[sys_pat].astype(np.int64)
        nf = plan.nfield[sys_pat].astype(np.int64)
        boff = np.concatenate([[0], np.cumsum(nd * nd)])
        hoff = np.concatenate([[0], np.cumsum(nd)])
        moff = np.concatenate([[0], np.cumsum(nf * nd)])
        fboff = np.concatenate([[0], np.cumsum(nf)])
        self.blocks = torch.empty(int(boff[-1]), dtype=torch.float64, device="cuda")
        self.hbar = torch.empty(int(hoff[-1]), dtype=torch.float64, device="cuda")
        self.M = torch.empty(int(moff[-1]) if keep_fields else 0, dtype=torch.float64,
                             device="cuda")
        self.Fb = torch.empty(int(fboff[-1]) if keep_fields else 0, dtype=torch.float64,
                              device="cuda")
        self.sys_boff, self.sys_hoff = boff[:-1], hoff[:-1]
        self.sys_moff, self.sys_fboff = moff[:-1], fboff[:-1]
        self.info = torch.zeros(nsys, dtype=torch.int32, device="cuda")
        work_d = np.array([pats[s].work_doubles for s, _ in systems], dtype=np.int64)
        x_d = np.array([pats[s].x_doubles for s, _ in systems], dtype=np.int64)
        smem = max(p.smem_doubles for p in pats)
        # waves bounded by the workspace budget
        per = 8 * (work_d + x_d)
        start = 0
        d_pat = _dev(sys_pat, torch.int32)
        d_koff = _dev(self.koff, torch.int64)
        d_boff, d_hoff = _dev(boff[:-1], torch.int64), _dev(hoff[:-1], torch.int64)
        d_moff, d_fboff = _dev(moff[:-1], torch.int64), _dev(fboff[:-1], torch.int64)
        phys = [plan.problem.layout.physics(s) for s, _ in systems]
        while start < nsys:
            end, acc = start, 0
            while end < nsys and (end == start or (acc + per[end] <= WORK_BUDGET_BYTES
                                                   and phys[end] == phys[start])):
                acc += per[end]
                end += 1
            cnt = end - start
            woff = np.concatenate([[0], np.cumsum(work_d[start:end])])
            xoff = np.concatenate([[0], np.cumsum(x_d[start:end])])
            work = torch.empty(int(woff[-1]), dtype=torch.float64, device="cuda")
            X = torch.empty(int(xoff[-1]), dtype=torch.float64, device="cuda")
            d_woff, d_xoff = _dev(woff[:-1], torch.int64), _dev(xoff[:-1], torch.int64)
            nt = threads or (512 if max(pats[s].kl for s, _ in systems[start:end]) > 128
                             else 256)
            sub = lambda t, elt=8: ctypes.c_void_p(t.data_ptr() + elt * start)
            if self.timing:
                e0 = self._ev()
            _lib.check(self.L.mfb_systems_solve(
                _ptr(plan.pat_dev), cnt, sub(d_pat, 4), _ptr(self.K), sub(d_koff),
                _ptr(work), _ptr(d_woff), _ptr(X), _ptr(d_xoff), sub(self.info, 4), nt, smem,
                self.sp), "mfb_systems_solve")
            if self.timing:
                self.solve_events.append((e0, self._ev()))
                self.solve_flops.append(sum(pats[s].algorithmic_flops for s, _ in
                                            systems[start:end]))
            self.launches += 2
            _lib.check(self.L.mfb_systems_extract(
                _ptr(plan.pat_dev), cnt, sub(d_pat, 4), _ptr(X), _ptr(d_xoff),
                _ptr(self.blocks), sub(d_boff), _ptr(self.hbar), sub(d_hoff),
                _ptr(self.M) if keep_fields else None, sub(d_moff),
                _ptr(self.Fb) if keep_fields else None, sub(d_fboff), self.sp),
                "mfb_systems_extract")
            start = end
        self.d_sys_moff, self.d_sys_fboff = d_moff, d_fboff
        # per-sid bases into the pool
        first = {}
        for idx, (s, l) in enumerate(systems):
            first.setdefault(s, idx)
        self.blk_base = np.array([boff[first[s]] for s in range(plan.n_sub)], dtype=np.int64)
        self.h_base = np.array([hoff[first[s]] for s in range(plan.n_sub)], dtype=np.int64)
        self.sys_first = first

    def check_info(self):
        info = self.info.cpu().numpy()
        bad = np.nonzero(info != 0)[0]
        if len(bad):
            s, l = self.systems[bad[0]]
            raise SingularOperatorError(
                f"subdomain {s} (local realization {l}): singular system "
                f"(device info {int(info[bad[0]])})")

    # ---------------------------------------------------------- (3) CG ----
    def solve_points(self, tol, max_iter, k0=0, n_pts=None, hist_cap=None, keep_g=False):
        torch, plan = self.torch, self.plan
        n_real = plan.grid.n_real
        n_pts = n_real - k0 if n_pts is None else n_pts
        nl = plan.n_lambda
        hist_cap = max_iter if hist_cap is None else hist_cap
        lam = torch.empty((n_pts, nl), dtype=torch.float64, device="cuda")
        iters = torch.empty(n_pts, dtype=torch.int32, device="cuda")
        status = torch.empty(n_pts, dtype=torch.int32, device="cuda")
        hist = torch.empty((n_pts, max(hist_cap, 1)), dtype=torch.float64, device="cuda")
        g = torch.empty((n_pts, nl), dtype=torch.float64, device="cuda") if keep_g else None
        d_blk, d_h = _dev(self.blk_base, torch.int64), _dev(self.h_base, torch.int64)
        self.launches += 1
        _lib.check(self.L.mfb_cg_batched(
            nl, plan.n_sub, _ptr(plan.d_ndof), _ptr(plan.d_dof_ptr), _ptr(plan.d_dof_map),
            _ptr(plan.d_region), _ptr(d_blk), _ptr(d_h), _ptr(plan.d_local), n_real,
            _ptr(self.blocks), _ptr(self.hbar), k0, n_pts, float(tol), int(max_iter),
            _ptr(lam), _ptr(iters), _ptr(status), _ptr(hist), max(hist_cap, 1),
            _ptr(g) if keep_g else None, self.sp), "mfb_cg_batched")
        return lam, iters, status, hist, g

    # ----------------------------------------------------- (4) moments ----
    def moments(self, lam):
        torch, plan = self.torch, self.plan
        grid = plan.grid
        nl, n_real = plan.n_lambda, grid.n_real
        out = {}
        m = torch.empty(nl, dtype=torch.float64, device="cuda")
        v = torch.empty_like(m)
        q = torch.empty_like(m)
        self.launches += 4
        _lib.check(self.L.mfb_lambda_moments(nl, n_real, _ptr(lam), _ptr(plan.d_weights),
                                             _ptr(m), _ptr(v), _ptr(q), self.sp),
                   "mfb_lambda_moments")
        # groups = systems; members from the region local-index tables
        systems = self.systems
        ng = len(systems)
        members, gptr = [], [0]
        order_cache = {}
        for s, l in systems:
            r = plan.region[s]
            if r < 0:
                mem = np.arange(n_real)
            else:
                if r not in order_cache:
                    li = grid.local_indices[r]
                    order = np.argsort(li, kind="stable")
                    bounds = np.searchsorted(li[order], np.arange(grid.local_counts[r] + 1))
                    order_cache[r] = (order, bounds)
                order, bounds = order_cache[r]
                mem = order[bounds[l]:bounds[l + 1]]
            members.append(mem)
            gptr.append(gptr[-1] + len(mem))
        grp_sid = np.array([s for s, _ in systems], dtype=np.int32)
        nd = plan.ndof[grp_sid].astype(np.int64)
        voff = np.concatenate([[0], np.cumsum(nd)])
        coff = np.concatenate([[0], np.cumsum(nd * nd)])
        d_sid = _dev(grp_sid, torch.int32)
        d_gptr = _dev(np.array(gptr), torch.int32)
        d_mem = _dev(np.concatenate(members), torch.int32)
        d_voff, d_coff = _dev(voff[:-1], torch.int64), _dev(coff[:-1], torch.int64)
        W = torch.empty(ng, dtype=torch.float64, device="cuda")
        lstar = torch.empty(int(voff[-1]), dtype=torch.float64, device="cuda")
        s_ = torch.empty_like(lstar)
        C = torch.empty(int(coff[-1]), dtype=torch.float64, device="cuda")
        _lib.check(self.L.mfb_group_stats(
            ng, _ptr(d_sid), _ptr(d_gptr), _ptr(d_mem), _ptr(plan.d_ndof), _ptr(plan.d_dof_ptr),
            _ptr(plan.d_dof_map), nl, _ptr(lam), _ptr(plan.d_weights), _ptr(d_voff),
            _ptr(d_coff), _ptr(W), _ptr(lstar), _ptr(s_), _ptr(C), self.sp), "mfb_group_stats")
        nfb = int(self.Fb.numel())
        fstar = torch.empty(nfb, dtype=torch.float64, device="cuda")
        t = torch.empty_like(fstar)
        qq = torch.empty_like(fstar)
        _lib.check(self.L.mfb_group_fields(
            ng, _ptr(d_sid), _ptr(plan.d_ndof), _ptr(plan.d_nfield), _ptr(self.M),
            _ptr(self.d_sys_moff), _ptr(self.Fb), _ptr(self.d_sys_fboff), _ptr(d_voff),
            _ptr(d_coff), _ptr(lstar), _ptr(s_), _ptr(C), _ptr(fstar), _ptr(t), _ptr(qq),
            self.sp), "mfb_group_fields")
        sid_gptr = np.array([self.sys_first[s] for s in range(plan.n_sub)] + [ng],
                            dtype=np.int32)
        out_off = np.concatenate([[0], np.cumsum(plan.nfield.astype(np.int64))])
        mean_f = torch.empty(int(out_off[-1]), dtype=torch.float64, device="cuda")
        var_f = torch.empty_like(mean_f)
        wtot = float(np.sum(grid.weights))
        d_sgptr = _dev(sid_gptr, torch.int32)
        d_outoff = _dev(out_off[:-1], torch.int64)
        _lib.check(self.L.mfb_moments_reduce(
            plan.n_sub, _ptr(d_sgptr), _ptr(plan.d_nfield),
            _ptr(self.d_sys_fboff), _ptr(W), _ptr(fstar), _ptr(t), _ptr(qq), wtot,
            _ptr(d_outoff), _ptr(mean_f), _ptr(var_f), self.sp),
            "mfb_moments_reduce")
        mh, vh, qh = m.cpu().numpy(), v.cpu().numpy(), q.cpu().numpy()
        out["lambda"] = _finalize("lambda", mh, vh, qh)
        mf, vf = mean_f.cpu().numpy(), var_f.cpu().numpy()
        for s in range(plan.n_sub):
            base = out_off[s]
            for name, start, shape in plan.patterns[s].field_layout:
                size = int(np.prod(shape))
                mm = mf[base + start: base + start + size].reshape(shape)
                vv = vf[base + start: base + start + size].reshape(shape)
                out[f"{s}:{name}"] = _finalize(f"{s}:{name}", mm, vv, vv + mm * mm)
        return out


def _finalize(key, mean, var, sumsq):
    """Clamp tiny negative variances like moments.py:43-58."""
    scale = max(1.0, float(np.max(np.abs(sumsq), initial=0.0)))
    bad = var < -1e-12 * scale
    if np.any(bad):
        log.warning("field %s: %d variance entries below -1e-12*scale (min %.3e), "
                    "clamping", key, int(np.sum(bad)), float(var.min()))
    return mean.copy(), np.maximum(var, 0.0)


def run_method(problem, grid, method="S1", tol=1e-9, max_iter=None, workers=1,
               basis_cap_mb=1024.0):
    """Sweep the collocation grid (reference interface.py:288-346), on the device.

    `workers` is accepted for signature compatibility; results do not depend
    on it (the device path is deterministic).
    """
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}, expected one of {METHODS}")
    if method != "S3":
        raise NotImplementedError(
            f"method {method} is not on this B200 path (S3 only); no CPU fallback")
    _lib.lib()                      # raises NativeLibraryError: no CPU fallback
    import torch
    t0 = time.perf_counter()
    n_sub = problem.layout.n_subdomains
    stats = SolveStats.new(method, n_sub)
    stats.n_real = grid.n_real
    nl = problem.space.n_dof
    if max_iter is None:
        max_iter = max(50, 10 * nl)
    plan = get_plan(problem, grid)
    _check_basis_cap(plan.basis_bytes(), basis_cap_mb)
    timings = {"plan": time.perf_counter() - t0}
    eng = S3Engine(plan)
    t1 = time.perf_counter()
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    torch.cuda.synchronize()
    timings["bases"] = time.perf_counter() - t1
    t2 = time.perf_counter()
    lam, iters, status, hist, _ = eng.solve_points(tol, max_iter)
    st = status.cpu().numpy()
    it = iters.cpu().numpy()
    timings["cg"] = time.perf_counter() - t2
    fail = np.nonzero((st == 1) | (st == 2))[0]
    hist_h = hist.cpu().numpy()
    if len(fail):
        k = int(fail[0])
        res = hist_h[k, :min(int(it[k]), hist_h.shape[1])].tolist()
        if st[k] == 1:
            raise ConvergenceError(f"interface operator is not positive definite "
                                   f"(p.Sp <= 0 at iteration {int(it[k])}, point {k})",
                                   res[:int(it[k]) - 1])
        raise ConvergenceError(f"CG did not reach tol {tol:g} in {max_iter} iterations "
                               f"(last residual {res[-1]:.3e}, point {k})", res)
    t3 = time.perf_counter()
    moments = eng.moments(lam)
    timings["moments"] = time.perf_counter() - t3
    lam_h = lam.cpu().numpy()
    lambdas = [lam_h[k] for k in range(grid.n_real)]
    residuals = [hist_h[k, :int(it[k])].tolist() for k in range(grid.n_real)]
    stats.cg_iters = [int(x) for x in it]
    for s in range(n_sub):
        nloc = int(plan.n_loc[s])
        stats.factorizations[s] = nloc
        stats.basis_backsolves[s] = int(plan.ndof[s]) * nloc
        stats.backsolves[s] = int(plan.ndof[s]) * nloc + 2 * grid.n_real
    stats.wall_seconds[:] = (time.perf_counter() - t0) / max(n_sub, 1)
    timings["total"] = time.perf_counter() - t0
    return RunResult(moments, stats, lambdas, residuals, grid, timings)
