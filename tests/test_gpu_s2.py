"""Method S2 (deterministic MFB) on the device vs the reference's own S2
sweep (tests/golden/make_golden_s2.py), and the S2-vs-S3 comparison that
BASELINE configs[1] asks for ("compare deterministic MFB and stochastic MFB
on identical inputs").

Tolerances as tests/test_gpu_parity.py: lambda and means 1e-8 relative at
CG tol 1e-11 (or 2x the reference's own reorder floor), variances 1e-8 or
2x the floor or |dvar| / max(mean^2) <= 1e-12.
"""

import numpy as np
import pytest

from conftest import FLOOR_MULT, case_from_golden, golden, iters_close

pytestmark = pytest.mark.gpu

TOL = 1e-11


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b))
                 / max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock", "case1_mini", "cfg2"])
def test_s2_sweep_matches_reference(gpu, name):
    from paper_1802_06263_b200.interface import run_method
    z = golden(name + "_s2")
    _, problem, grid, _ = case_from_golden(name)
    res = run_method(problem, grid, method="S2", tol=TOL)
    L = np.array(res.lambdas)
    assert _rel(L, z["s2_lambda"]) <= max(1e-8, FLOOR_MULT * float(z["floor_lambda"]))
    for key in res.moments:
        m, v = res.moments[key]
        mg, vg = z[f"mean__{key}"], z[f"var__{key}"]
        assert m.shape == mg.shape and v.shape == vg.shape, key
        fm = float(z[f"floor_mean__{key}"])
        assert (_rel(m, mg) <= max(1e-8, FLOOR_MULT * fm)
                or np.max(np.abs(m - mg)) <= 1e-12), (key, _rel(m, mg), fm)
        fv = float(z[f"floor_var__{key}"])
        scale = max(float(np.max(mg * mg)), 1e-300)
        assert (_rel(v, vg) <= max(1e-8, FLOOR_MULT * fv)
                or np.max(np.abs(v - vg)) / scale <= 1e-12), (key, _rel(v, vg), fv)
    it = np.array(res.stats.cg_iters)
    itg = z["s2_iters"]
    assert iters_close(it.mean(), itg.mean())
    # counters in the reference's S2 semantics (one factorization and
    # N_dof + 2 backsolves per subdomain per realization)
    assert list(res.stats.factorizations) == list(z["stats_factorizations"])
    assert list(res.stats.basis_backsolves) == list(z["stats_basis_backsolves"])
    assert list(res.stats.backsolves) == list(z["stats_backsolves"])


def test_s2_equals_s3_when_stokes_is_decoupled(gpu):
    """alpha = 0 removes the only K dependence of the Stokes operator (the BJS
    term), so S3's frozen Stokes blocks equal S2's per-realization ones and
    the Darcy blocks are the same local realizations: the two methods give
    the same sweep (the reference's CRITERION, test_acceptance.py:124-141)."""
    from paper_1802_06263_b200.interface import run_method
    _, problem, grid, _ = case_from_golden("cfg2", physics={"alpha": 0.0, "nu_s": 1.0, "nu_d": 1.0})
    r2 = run_method(problem, grid, method="S2", tol=TOL)
    r3 = run_method(problem, grid, method="S3", tol=TOL)
    assert _rel(np.array(r2.lambdas), np.array(r3.lambdas)) <= 1e-8
    for key in r3.moments:
        assert _rel(r2.moments[key][0], r3.moments[key][0]) <= 1e-8 or \
            np.max(np.abs(r2.moments[key][0] - r3.moments[key][0])) <= 1e-12, key


def test_s2_s3_blocks_share_darcy_realizations(gpu):
    """S2's Darcy block of realization k is S3's block of loc_i(k) (same K,
    same kernel): bitwise, as the reference's S3 == S2 check
    (test_interface.py:129-140) relies on."""
    from paper_1802_06263_b200.interface import SweepEngine, get_plan
    _, problem, grid, _ = case_from_golden("cfg1")
    plan = get_plan(problem, grid)
    e3 = SweepEngine(plan, method="S3")
    e3.kl_fields(); e3.build_bases(); e3.check_info()
    b3 = e3.blocks.cpu().numpy()
    e2 = SweepEngine(plan, method="S2")
    e2.kl_fields(); e2.build_bases(); e2.check_info()
    b2 = e2.blocks.cpu().numpy()
    sys3 = {sl: i for i, sl in enumerate(e3.systems)}
    checked = 0
    for i, (s, k) in enumerate(e2.systems):
        if plan.region[s] < 0:
            continue
        loc = int(grid.local_indices[plan.region[s]][k])
        j = sys3[(s, loc)]
        nd = int(plan.ndof[s])
        a = b2[e2.sys_boff[i]: e2.sys_boff[i] + nd * nd]
        b = b3[e3.sys_boff[j]: e3.sys_boff[j] + nd * nd]
        assert np.array_equal(a, b), (s, k)
        checked += 1
    assert checked > 0


def test_methods_and_size_cap_errors(gpu):
    """run_method's error conventions (interface.py:288-346): unknown method
    -> ValueError; the basis-memory cap -> SizeCapError before any device
    work, checked on the whole S3 pool (interface.py:375) but on ONE
    realization's bases for S2 (interface.py:320-322); S1 stores no basis
    and ignores the cap."""
    from paper_1802_06263_b200.errors import SizeCapError
    from paper_1802_06263_b200.interface import get_plan, run_method
    _, problem, grid, _ = case_from_golden("cfg2")
    with pytest.raises(ValueError):
        run_method(problem, grid, method="S4")
    plan = get_plan(problem, grid)
    s3_mb = sum(plan.basis_bytes("S3")) / 2 ** 20
    s2_mb = sum(plan.basis_bytes("S2")) / 2 ** 20
    assert s2_mb < s3_mb
    with pytest.raises(SizeCapError):
        run_method(problem, grid, method="S3", tol=TOL, basis_cap_mb=0.5 * s3_mb)
    with pytest.raises(SizeCapError):
        run_method(problem, grid, method="S2", tol=TOL, basis_cap_mb=0.5 * s2_mb)
    # a cap between the two: S2 (one realization at a time in the reference's
    # accounting) runs, S3 (the whole local pool) does not
    cap = 0.5 * (s2_mb + s3_mb)
    res = run_method(problem, grid, method="S2", tol=TOL, basis_cap_mb=cap)
    assert len(res.lambdas) == grid.n_real
    with pytest.raises(SizeCapError):
        run_method(problem, grid, method="S3", tol=TOL, basis_cap_mb=cap)


def test_in_place_problem_changes_rebuild_the_plan(gpu):
    """The reference's problem is a mutable dataclass: swapping its physics in
    place between two run_method calls must not reuse the resident plan
    built for the old physics."""
    import dataclasses
    from paper_1802_06263_b200.interface import run_method
    _, problem, grid, _ = case_from_golden("cfg1")
    r1 = run_method(problem, grid, method="S3", tol=TOL)
    problem.physics = dataclasses.replace(problem.physics, alpha=0.0)
    r2 = run_method(problem, grid, method="S3", tol=TOL)
    _, fresh, grid0, _ = case_from_golden("cfg1", physics={"alpha": 0.0})
    r3 = run_method(fresh, grid0, method="S3", tol=TOL)
    assert not np.array_equal(np.array(r1.lambdas), np.array(r2.lambdas))
    assert np.array_equal(np.array(r2.lambdas), np.array(r3.lambdas))
