"""Multi-GPU S3 sweep: one process per GPU, torch.distributed for the plumbing.

The path shards naturally:

* pre-loop: subdomains are assigned to ranks (`sid_owners`); a rank builds
  the flux-basis blocks, bar jumps and field responses of its subdomains'
  local realizations only, then one all-reduce (SUM over zero-padded pools,
  exact because every slot has a single non-zero contributor) gives every
  rank the full basis pool;
* main loop: each rank runs the batched CG on an interleaved set of
  collocation points (`point_set`: k = rank mod world); one all-gather
  assembles lambda in point order;
* moments: the rank that owns a subdomain reduces its field keys with the
  exact single-GPU arithmetic (groups live with their subdomain), rank 0
  streams the lambda key; results are gathered on rank 0 in key order.

Every number a rank computes is computed by the same kernel with the same
inputs as on one GPU, so the N-rank result is bitwise the 1-rank result.
The collectives are ordinary torch.distributed calls (NCCL on GPUs, gloo in
the CPU tests), and `Engine` is the device engine (`interface.SweepEngine`) or
a CPU stand-in used by tests/test_distributed.py. Verdicts are collective: a
singular system on any rank raises SingularOperatorError on every rank
(agreed before the first data collective), a failed point raises
ConvergenceError on every rank (all ranks hold the gathered statuses).
"""

import numpy as np


def point_range(n_real, rank, world):
    """Contiguous [k0, k1) block of collocation points for one rank."""
    base, extra = divmod(n_real, world)
    k0 = rank * base + min(rank, extra)
    return k0, k0 + base + (1 if rank < extra else 0)


def point_set(n_real, rank, world):
    """The collocation points of one rank: k = rank (mod world). Interleaved,
    not contiguous: a point's CG iteration count is not known in advance
    (13k-75k at cfg4) and neighbouring Smolyak points are alike, so the
    interleaving balances the ranks' work."""
    return np.arange(rank, n_real, world, dtype=np.int64)


def sid_owners(costs, world):
    """Greedy longest-processing-time assignment of subdomains to ranks.

    `costs[s]` is the basis-construction cost of subdomain s (systems x
    work); ties go to the lowest rank, so the assignment is deterministic.
    """
    order = sorted(range(len(costs)), key=lambda s: (-costs[s], s))
    load = [0.0] * world
    owner = [0] * len(costs)
    for s in order:
        r = min(range(world), key=lambda q: (load[q], q))
        owner[s] = r
        load[r] += costs[s]
    return owner


def agree_error(err, dist, world):
    """Collective verdict: every rank learns whether any rank failed and the
    first failing rank's message (so all raise together; a rank raising alone
    before a collective would leave the others waiting in it)."""
    msgs = [None] * world
    dist.all_gather_object(msgs, err)
    return next((m for m in msgs if m is not None), None)


def run_sharded(engine, n_real, n_lambda, tol, max_iter, dist, rank, world):
    """Drive one sharded sweep; returns (moments, lam, iters, status, hist) on
    every rank (moments merged on rank 0, None elsewhere).

    engine: object with build(sids) -> None or an error message (a singular
    system), pools() -> list of tensors to all-reduce, solve(points, tol,
    max_iter) -> (lam, iters, status, hist), moments(lam_all, sids,
    with_lambda) -> dict, to_host(t) -> numpy, and torch-like tensors.
    dist: torch.distributed (initialised). Raises SingularOperatorError on
    every rank when any rank's systems are singular.
    """
    import torch

    from .errors import SingularOperatorError
    owners = sid_owners(engine.sid_costs(), world)
    mine = [s for s, r in enumerate(owners) if r == rank]
    err = agree_error(engine.build(mine), dist, world)
    if err is not None:
        raise SingularOperatorError(err)
    for t in engine.pools():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    pts = point_set(n_real, rank, world)
    lam, iters, status, hist = engine.solve(pts, tol, max_iter)
    dev = lam.device
    width = len(point_set(n_real, 0, world))
    hcols = torch.tensor([hist.shape[1]], dtype=torch.int64, device=dev)
    dist.all_reduce(hcols, op=dist.ReduceOp.MAX)
    hcols = int(hcols.item())

    def gather(x, cols, dtype):
        """rows of every rank's points, placed at their global indices"""
        buf = torch.zeros((width, cols), dtype=dtype, device=dev)
        xx = x.reshape(x.shape[0], -1)
        buf[:xx.shape[0], :xx.shape[1]] = xx
        out = [torch.zeros_like(buf) for _ in range(world)]
        dist.all_gather(out, buf)
        full = torch.zeros((n_real, cols), dtype=dtype, device=dev)
        for r in range(world):
            idx = torch.as_tensor(point_set(n_real, r, world), device=dev)
            full[idx] = out[r][:len(idx)]
        return full

    lam_all = gather(lam, n_lambda, lam.dtype)
    iters_all = gather(iters.to(torch.int64), 1, torch.int64).reshape(-1)
    status_all = gather(status.to(torch.int64), 1, torch.int64).reshape(-1)
    hist_all = gather(hist, hcols, hist.dtype)
    mom = engine.moments(lam_all, mine, with_lambda=(rank == 0))
    gathered = [None] * world
    dist.all_gather_object(gathered, mom)
    moments = None
    if rank == 0:
        merged = {}
        for part in gathered:
            merged.update(part)
        keys = ["lambda"] + sorted((k for k in merged if k != "lambda"),
                                   key=lambda k: (int(k.split(":")[0]),
                                                  ["u", "p", "cv", "cp"].index(k.split(":")[1])))
        moments = {k: merged[k] for k in keys}
    return (moments, engine.to_host(lam_all), engine.to_host(iters_all),
            engine.to_host(status_all), engine.to_host(hist_all))


class DeviceShardEngine:
    """`run_sharded` engine over the sm_100a SweepEngine (one GPU per rank)."""

    def __init__(self, plan):
        from .interface import SweepEngine
        self.plan = plan
        self.eng = SweepEngine(plan)

    def sid_costs(self):
        p = self.plan
        return [float(int(p.n_loc[s]) * (p.hyb[s].algorithmic_flops if s in p.hyb
                                           else p.patterns[s].algorithmic_flops))
                for s in range(p.n_sub)]

    def build(self, sids):
        """This rank's systems; None, or the message of its first singular
        system (raised by run_sharded on every rank, after agreement)."""
        from .errors import SingularOperatorError
        st = self.eng.st
        st.blocks.zero_()
        st.hbar.zero_()
        self.eng.kl_fields()
        self.eng.build_bases(sids=sids)
        try:
            self.eng.check_info()
        except SingularOperatorError as e:
            return str(e)
        return None

    def pools(self):
        return [self.eng.st.blocks, self.eng.st.hbar]

    def solve(self, pts, tol, max_iter):
        """CG of the points `pts` (global indices): the kernels see them as
        points 0..n-1 of a local-index table gathered for this rank."""
        import torch

        from .interface import hist_padded
        table = self.eng.st.d_cg_local[:, torch.as_tensor(pts, device="cuda")].contiguous()
        lam, iters, status, hist, _ = self.eng.solve_points(
            tol, max_iter, k0=0, n_pts=len(pts), local_override=table)
        return lam, iters, status, hist_padded(hist, iters)

    def moments(self, lam_all, sids, with_lambda):
        return self.eng.moments(lam_all, sids=sids, with_lambda=with_lambda)

    @staticmethod
    def to_host(t):
        return t.cpu().numpy()


def run_method_distributed(problem, grid, tol=1e-9, max_iter=None, basis_cap_mb=1024.0):
    """S3 sweep sharded over the initialised torch.distributed world.

    Returns the RunResult on rank 0 and None elsewhere.
    """
    import torch.distributed as dist

    from .errors import ConvergenceError
    from .interface import RunResult, SolveStats, _check_basis_cap, get_plan
    rank, world = dist.get_rank(), dist.get_world_size()
    plan = get_plan(problem, grid)
    _check_basis_cap(plan.basis_bytes(), basis_cap_mb)
    nl = problem.space.n_dof
    if max_iter is None:
        max_iter = max(50, 10 * nl)
    moments, lam, iters, status, hist = run_sharded(DeviceShardEngine(plan), grid.n_real, nl,
                                                    tol, max_iter, dist, rank, world)
    # every rank holds the gathered verdicts: all raise together
    fail = np.nonzero((status == 1) | (status == 2))[0]
    if len(fail):
        k = int(fail[0])
        raise ConvergenceError(f"CG failed at point {k} (status {int(status[k])})",
                               hist[k, :int(iters[k])].tolist())
    if rank != 0:
        return None
    stats = SolveStats.new("S3", plan.n_sub)
    stats.n_real = grid.n_real
    stats.cg_iters = [int(x) for x in iters]
    for s in range(plan.n_sub):
        nloc = int(plan.n_loc[s])
        stats.factorizations[s] = nloc
        stats.basis_backsolves[s] = int(plan.ndof[s]) * nloc
        stats.backsolves[s] = int(plan.ndof[s]) * nloc + 2 * grid.n_real
    return RunResult(moments, stats, [lam[k] for k in range(grid.n_real)],
                     [hist[k, :int(iters[k])].tolist() for k in range(grid.n_real)], grid)
