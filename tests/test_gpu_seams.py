"""The reference's secondary seams on the device (paper_1802_06263_b200/seams.py)
against the reference's own functions (sdmortar.interface) on the same
inputs: solve_realization (interface.py:417-437), basis_apply (238-247),
cg_solve (107-139, every status path) and compute_flux_basis (218-235)."""

import numpy as np
import pytest

from conftest import case_from_golden, iters_close


def _rel(a, b):
    a, b = np.asarray(a, dtype=float).ravel(), np.asarray(b, dtype=float).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["darcy_twoblock", "cfg1"])
def test_solve_realization_matches_reference(gpu, name):
    import sdmortar.interface as ri
    from paper_1802_06263_b200 import seams
    _, problem, grid, _ = case_from_golden(name)
    for y in (None, grid.points[len(grid.points) // 2]):
        ref_f, ref_lam, ref_st = ri.solve_realization(problem, y, tol=1e-11)
        f, lam, st = seams.solve_realization(problem, y, tol=1e-11)
        assert _rel(lam, ref_lam) <= 1e-8
        assert len(f) == len(ref_f)
        for a, b in zip(f, ref_f):
            assert sorted(a) == sorted(b)
            for k in b:
                assert np.asarray(a[k]).shape == np.asarray(b[k]).shape
                assert _rel(a[k], b[k]) <= 1e-8 or np.max(np.abs(a[k] - b[k])) <= 1e-12, k
        # (symmetrised device blocks: a few iterations fewer, conftest.iters_close)
        assert st.n_real == 1 and iters_close(st.cg_iters[0], ref_st.cg_iters[0])
        assert list(st.factorizations) == list(ref_st.factorizations)


@pytest.mark.gpu
def test_basis_apply_and_cg_solve_match_reference(gpu):
    import sdmortar.interface as ri
    from sdmortar.errors import ConvergenceError
    from paper_1802_06263_b200 import seams
    _, problem, grid, _ = case_from_golden("cfg1")
    n_sub = problem.layout.n_subdomains
    stats = ri.SolveStats.new("S3", n_sub)
    K = problem.permeability(np.zeros(grid.n_dims))
    ops = [problem.assemble_subdomain(s, K) for s in range(n_sub)]
    bases = [ri.compute_flux_basis(problem, s, ops[s], stats) for s in range(n_sub)]
    dev, ref = seams.basis_apply(problem.space, bases), ri.basis_apply(problem.space, bases)
    rng = np.random.default_rng(5)
    v = rng.standard_normal(problem.space.n_dof)
    assert _rel(dev(v), ref(v)) <= 1e-13
    g = rng.standard_normal(problem.space.n_dof)
    x, it, res = seams.cg_solve(dev, g, tol=1e-11)
    xr, itr, resr = ri.cg_solve(ref, g, tol=1e-11)
    assert _rel(x, xr) <= 1e-8 and abs(it - itr) <= 2 and len(res) == it
    assert res[-1] <= 1e-11 and abs(res[0] - resr[0]) <= 1e-12 * max(1.0, resr[0])
    # zero rhs: no iterations (interface.py:111-113)
    x0, it0, res0 = seams.cg_solve(dev, np.zeros_like(g))
    assert it0 == 0 and res0 == [] and not np.any(x0)
    # budget exhausted: ConvergenceError with the residual history
    with pytest.raises(ConvergenceError) as e:
        seams.cg_solve(dev, g, tol=1e-14, max_iter=3)
    assert len(e.value.residuals) == 3
    # not positive definite (negated blocks)
    neg = seams.basis_apply(problem.space, [(d, -B) for d, B in bases])
    with pytest.raises(ConvergenceError):
        seams.cg_solve(neg, g)
    # a plain callable is the reference's host CG, unchanged
    A = np.diag(np.arange(1.0, 6.0))
    xh, ith, _ = seams.cg_solve(lambda w: A @ w, np.ones(5), tol=1e-12)
    assert np.allclose(A @ xh, np.ones(5)) and ith <= 5


@pytest.mark.gpu
def test_compute_flux_basis_matches_reference(gpu):
    import sdmortar.interface as ri
    from paper_1802_06263_b200 import seams
    _, problem, grid, _ = case_from_golden("cfg1")
    n_sub = problem.layout.n_subdomains
    y = grid.points[3]
    K = problem.permeability(y)
    for sid in range(n_sub):
        st_r, st_d = ri.SolveStats.new("S3", n_sub), ri.SolveStats.new("S3", n_sub)
        dofs_r, B_r = ri.compute_flux_basis(problem, sid, problem.assemble_subdomain(sid, K), st_r)
        dofs_d, B_d = seams.compute_flux_basis(problem, sid, seams.assemble_subdomain(problem, sid, K),
                                               st_d)
        assert np.array_equal(np.asarray(dofs_d), np.asarray(dofs_r))
        assert np.max(np.abs(B_d - B_r)) <= 1e-10 * np.max(np.abs(B_r)), sid
        assert st_d.basis_backsolves[sid] == st_r.basis_backsolves[sid]
