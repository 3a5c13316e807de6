"""Device edge cases through the C ABI: the banded solver on synthetic
systems (pivoting, cooperative groups, zero pivots that must end every CTA
of the group), the batched CG's status paths (zero rhs, breakdown, budget),
empty launches, and the reference's ConvergenceError semantics."""
import ctypes

import numpy as np
import pytest

from conftest import case_from_golden

pytestmark = pytest.mark.gpu


def _dev(a, dtype):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a), dtype=dtype).to("cuda")


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def _band_system(n, kl, ku, seed, zero_col=None):
    """Random banded matrix with weak diagonals (partial pivoting is needed),
    entries listed like a Pattern (constant terms)."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - kl), min(n, i + ku + 1)):
            A[i, j] = rng.uniform(-1, 1)
        A[i, i] *= 0.05                      # small diagonal: row swaps happen
    if zero_col is not None:
        A[:, zero_col] = 0.0
    r, c = np.nonzero(A)
    return A, r.astype(np.int32), c.astype(np.int32), A[r, c]


def _solve_band(A, rows, cols, vals, kl, ku, rhs, group):
    import torch

    from paper_1802_06263_b200 import _lib
    from paper_1802_06263_b200.discretization import Pattern
    n, ndof = A.shape[0], rhs.shape[1] - 1
    i32, f64 = torch.int32, torch.float64
    ne = len(rows)
    q_ptr = np.arange(0, n * ndof + 1, n, dtype=np.int32)          # dense Q columns
    q_row = np.tile(np.arange(n, dtype=np.int32), ndof)
    q_val = rhs[:, :ndof].T.ravel()
    keep = dict(
        e_row=_dev(rows, i32), e_col=_dev(cols, i32), e_tptr=_dev(np.arange(ne + 1), i32),
        t_kind=_dev(np.zeros(ne), i32), t_c=_dev(vals, f64), t_k=_dev(np.zeros(ne), i32),
        q_ptr=_dev(q_ptr, i32), q_row=_dev(q_row, i32), q_val=_dev(q_val, f64),
        bar_const=_dev(rhs[:, ndof], f64))
    st = _lib.MfbPattern()
    st.n, st.kl, st.ku, st.ldab, st.nb, st.ndof, st.nfield = n, kl, ku, 2 * kl + ku + 1, 0, ndof, 0
    st.n_entries, st.n_bar_rows = ne, 0
    for k, t in keep.items():
        setattr(st, k, _ptr(t).value or 0)
    pats = torch.frombuffer(bytearray(bytes(st)), dtype=torch.uint8).to("cuda")
    host = Pattern(0, "test", n, kl, ku, 0, ndof, 0, *([np.zeros(1)] * 22))
    K = torch.ones(1, dtype=f64, device="cuda")
    work = torch.zeros(host.work_doubles, dtype=f64, device="cuda")
    X = torch.zeros(n * (ndof + 1), dtype=f64, device="cuda")
    zero64 = torch.zeros(1, dtype=torch.int64, device="cuda")
    info = torch.full((1,), -99, dtype=i32, device="cuda")
    bar = torch.zeros(2, dtype=i32, device="cuda")
    sys_pat = torch.zeros(1, dtype=i32, device="cuda")
    L = _lib.lib()
    _lib.check(L.mfb_systems_solve(_ptr(pats), 1, _ptr(sys_pat), _ptr(K), _ptr(zero64),
                                   _ptr(work), _ptr(zero64), _ptr(X), _ptr(zero64), _ptr(info),
                                   256, host.smem_doubles, group, _ptr(bar), 0, None),
               "mfb_systems_solve")
    torch.cuda.synchronize()
    return X.cpu().numpy().reshape(n, ndof + 1), int(info.item())


@pytest.mark.timeout(120)
@pytest.mark.parametrize("group", [1, 2, 5])
def test_band_solver_random_pivoting_system(gpu, group):
    n, kl, ku = 203, 21, 17                      # ragged last panel, kl != ku
    A, r, c, v = _band_system(n, kl, ku, seed=group)
    rhs = np.random.default_rng(9).standard_normal((n, 4))
    X, info = _solve_band(A, r, c, v, kl, ku, rhs, group)
    assert info == 0
    ref = np.linalg.solve(A, rhs)
    assert np.max(np.abs(X - ref)) / np.max(np.abs(ref)) <= 1e-10


@pytest.mark.timeout(120)
@pytest.mark.parametrize("group", [1, 3])
def test_band_solver_zero_pivot_ends_every_cta(gpu, group):
    """A zero column must report info = j + 1 and finish (no CTA of the
    cooperative group may keep waiting for a panel that never comes)."""
    n, kl, ku = 160, 12, 12
    A, r, c, v = _band_system(n, kl, ku, seed=4, zero_col=77)
    rhs = np.ones((n, 2))
    _, info = _solve_band(A, r, c, v, kl, ku, rhs, group)
    assert info == 78


def _cg(blocks, hbar, nd, n_lambda, max_iter, tol=1e-12, stage=True, regs=False):
    import torch

    from paper_1802_06263_b200 import _lib
    i32, i64, f64 = torch.int32, torch.int64, torch.float64
    n_sub = len(nd)
    dof_ptr = np.concatenate([[0], np.cumsum(nd)]).astype(np.int32)
    dof_map = np.concatenate([np.arange(k) for k in nd]).astype(np.int32)
    blk_base = np.concatenate([[0], np.cumsum([k * k for k in nd])[:-1]]).astype(np.int64)
    h_base = dof_ptr[:-1].astype(np.int64)
    t = {k: _dev(a, dt) for k, (a, dt) in dict(
        ndof=(np.array(nd), i32), dof_ptr=(dof_ptr, i32), dof_map=(dof_map, i32),
        region=(np.full(n_sub, -1), i32), blk=(blk_base, i64), h=(h_base, i64),
        loc=(np.zeros(1), i32), blocks=(blocks, f64), hbar=(hbar, f64)).items()}
    lam = torch.zeros(n_lambda, dtype=f64, device="cuda")
    iters = torch.zeros(1, dtype=i32, device="cuda")
    status = torch.full((1,), -1, dtype=i32, device="cuda")
    hist = torch.zeros(max(max_iter, 1), dtype=f64, device="cuda")
    L = _lib.lib()
    _lib.check(L.mfb_cg_batched(
        n_lambda, n_sub, _ptr(t["ndof"]), _ptr(t["dof_ptr"]), _ptr(t["dof_map"]),
        _ptr(t["region"]), _ptr(t["blk"]), _ptr(t["h"]), _ptr(t["loc"]), 1, _ptr(t["blocks"]),
        _ptr(t["hbar"]), 0, 1, tol, max_iter, _ptr(lam), _ptr(iters), _ptr(status), _ptr(hist),
        max(max_iter, 1), None, int(sum(k * k for k in nd)) if stage else 0,
        max(nd) if regs and all(k % 4 == 0 for k in nd) else 0, None),
        "mfb_cg_batched")
    torch.cuda.synchronize()
    return lam.cpu().numpy(), int(iters.item()), int(status.item()), hist.cpu().numpy()


@pytest.mark.parametrize("stage,regs", [(True, False), (False, False), (False, True)])
def test_cg_status_paths(gpu, stage, regs):
    """Staged blocks, blocks read from L2, and block rows in registers (the
    latter needs ndof % 4 == 0)."""
    rng = np.random.default_rng(3)
    nl = 8 if regs else 5
    nd = [nl, nl]                                  # two sides of every dof
    M1 = rng.standard_normal((nl, nl))
    M2 = rng.standard_normal((nl, nl))
    B1, B2 = M1 @ M1.T + nl * np.eye(nl), M2 @ M2.T + nl * np.eye(nl)
    blocks = np.concatenate([B1.T.ravel(), B2.T.ravel()])    # column-major storage
    h = rng.standard_normal(2 * nl)
    # converged, against a dense solve of (B1 + B2) lam = h1 + h2
    lam, it, status, hist = _cg(blocks, h, nd, nl, 50, stage=stage, regs=regs)
    ref = np.linalg.solve(B1 + B2, h[:nl] + h[nl:])
    assert status == 0 and 1 <= it <= 50
    assert np.max(np.abs(lam - ref)) / np.max(np.abs(ref)) <= 1e-10
    assert hist[it - 1] <= 1e-12
    # zero rhs: no iterations, lambda = 0 (interface.py:111-113)
    lam, it, status, _ = _cg(blocks, np.zeros(2 * nl), nd, nl, 50, stage=stage, regs=regs)
    assert status == 3 and it == 0 and not lam.any()
    # breakdown on a negative definite operator (interface.py:123-126)
    _, it, status, _ = _cg(-blocks, h, nd, nl, 50, stage=stage, regs=regs)
    assert status == 1 and it == 1
    # budget exhausted (interface.py:137-139)
    _, it, status, hist = _cg(blocks, h, nd, nl, 2, stage=stage, regs=regs)
    assert status == 2 and it == 2 and hist[1] > 1e-12


def test_empty_launches_are_noops(gpu):
    from paper_1802_06263_b200 import _lib
    L = _lib.lib()
    z = ctypes.c_void_p(0)
    assert L.mfb_systems_solve(z, 0, z, z, z, z, z, z, z, z, 256, 0, 1, z, 0, None) == 0
    assert L.mfb_cg_batched(4, 1, z, z, z, z, z, z, z, 1, z, z, 0, 0, 1e-9, 10, z, z, z, z, 1,
                            z, 0, 0, None) == 0
    assert L.mfb_systems_solve(z, -1, z, z, z, z, z, z, z, z, 256, 0, 1, z, 0, None) == 1


def test_run_method_raises_convergence_error_with_history(gpu):
    from paper_1802_06263_b200.errors import ConvergenceError
    from paper_1802_06263_b200.interface import run_method
    _, problem, grid, _ = case_from_golden("cfg1")
    with pytest.raises(ConvergenceError) as e:
        run_method(problem, grid, method="S3", tol=1e-11, max_iter=3)
    assert len(e.value.residuals) == 3


@pytest.mark.gpu
def test_shape_limits_raise_instead_of_overrunning(gpu):
    """The device kernels' fixed shape limits fail loudly:
    a KL region with more than 64 terms (mfb_kl_realize_batched stages xi in
    64 shared doubles) and a subdomain with more than 64 mortar dofs (the
    moment kernels' block tiles) raise NativeLibraryError before any launch
    that would overrun."""
    from paper_1802_06263_b200.errors import NativeLibraryError
    from paper_1802_06263_b200.interface import run_method
    many_terms = {"kl_regions": [{"eta": [0.4, 0.4], "n_term": 72, "rect": [0.0, 0.0, 2.0, 1.0],
                                  "selection": "largest", "sigma2": 0.5}],
                  "collocation": {"kind": "tensor", "m": 1}}
    _, problem, grid, _ = case_from_golden("darcy_twoblock", **many_terms)
    with pytest.raises(NativeLibraryError, match="KL"):
        run_method(problem, grid, method="S3", tol=1e-9)
    wide = {"mortars": {"allow_fine": True, "dd": 72, "degree": 0, "per_interface": {}}}
    _, problem, grid, _ = case_from_golden("darcy_twoblock", **wide)
    assert max(len(problem.space.sub_dofs(problem.layout, s)) for s in range(2)) > 64
    with pytest.raises(NativeLibraryError, match="mortar dofs"):
        run_method(problem, grid, method="S3", tol=1e-9)


def test_wall_seconds_are_measured_per_subdomain(gpu):
    """SolveStats.wall_seconds (interface.py:142-154: per-subdomain assembly,
    bases, bar solves, recovery): the measured device time of each
    subdomain's basis systems, not the call's time divided evenly."""
    from paper_1802_06263_b200.interface import run_method
    _, problem, grid, _ = case_from_golden("cfg2")
    res = run_method(problem, grid, method="S3", tol=1e-11)
    ws = np.asarray(res.stats.wall_seconds)
    assert ws.shape == (problem.layout.n_subdomains,)
    assert np.all(np.isfinite(ws)) and np.all(ws > 0.0)
    phys = np.array([problem.layout.physics(s) for s in range(len(ws))])
    # Stokes and Darcy subdomains run different kernels: their times differ
    assert abs(ws[phys == "stokes"].mean() - ws[phys == "darcy"].mean()) > 0.0
    assert len(np.unique(np.round(ws, 12))) > 1
    # every wave is counted once: the sum stays within the device time of
    # the call (two overlapping streams can double the basis phase at most)
    assert ws.sum() <= 2.0 * res.timings["device"] + 1e-3
    rows = res.stats.rows()
    assert all(r["wall_seconds"] == float(ws[r["subdomain"]]) for r in rows)
