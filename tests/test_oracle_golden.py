"""Pin the CPU oracle (oracle/s3_cpu.py) against the reference's own outputs.

The golden fixtures were produced by running the reference package
(tests/golden/make_golden.py). The oracle restates the same algorithm
(SuperLU factor, per-dof star solves, numpy CG), so basis blocks agree to
roundoff and sweeps agree at the reference's own reorder noise floor.
"""

import numpy as np
import pytest

from conftest import case_from_golden, golden

TOL = 1e-11


def _rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) /
                 max(np.linalg.norm(np.ravel(b)), 1e-300))


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock", "case1_mini", "cfg2"])
def test_oracle_sweep_matches_reference(name):
    from oracle import s3_cpu
    z = golden(name)
    _, problem, grid, _ = case_from_golden(name)
    r = s3_cpu.run_s3(problem, grid, tol=TOL, record_g=True)
    for sid, bl in r["bases"].items():
        for loc, (_, B) in enumerate(bl):
            key = f"B__{sid}__{loc}"
            if key in z:
                assert np.max(np.abs(B - z[key])) <= 1e-11 * np.max(np.abs(z[key])), key
    assert np.max(np.abs(np.array(r["g"]) - z["s3_g"])) <= 1e-11 * np.max(np.abs(z["s3_g"]))
    assert _rel(np.array(r["lambdas"]), z["s3_lambda"]) <= 1e-9
    for key, (m, v) in r["moments"].items():
        assert _rel(m, z[f"mean__{key}"]) <= 1e-8 or np.max(np.abs(m - z[f"mean__{key}"])) <= 1e-12
        floor = float(z[f"floor_var__{key}"])
        vg = z[f"var__{key}"]
        scale = max(float(np.max(z[f"mean__{key}"] ** 2)), 1e-300)
        assert _rel(v, vg) <= max(1e-8, 10 * floor) or np.max(np.abs(v - vg)) / scale <= 1e-12


def test_oracle_known_answer_uniform_flow():
    """K = 1 two-block Darcy: lambda = 0.5, linear pressure (test_interface.py:53-62)."""
    from oracle import s3_cpu
    _, problem, grid, _ = case_from_golden(
        "darcy_twoblock", collocation={"kind": "tensor", "m": 1})
    r = s3_cpu.run_s3(problem, grid, tol=1e-12)
    assert np.allclose(r["lambdas"][0], 0.5, atol=1e-9)
    m, _ = r["moments"]["0:cv"]
    assert np.allclose(m[:, 0], 0.5, atol=1e-9) and np.allclose(m[:, 1], 0.0, atol=1e-9)
    xc = problem.meshes[0].centroids[:, 0]
    assert np.allclose(r["moments"]["0:cp"][0], 1.0 - xc / 2.0, atol=1e-9)


def test_oracle_cg_error_paths():
    from oracle.s3_cpu import cg_solve
    from paper_1802_06263_b200.errors import ConvergenceError
    x, it, res = cg_solve(lambda v: v, np.zeros(5))
    assert it == 0 and res == [] and not x.any()
    with pytest.raises(ConvergenceError, match="positive definite"):
        cg_solve(lambda v: -v, np.ones(4))
    A = np.diag(np.linspace(1.0, 1e4, 30))
    with pytest.raises(ConvergenceError) as err:
        cg_solve(lambda v: A @ v, np.ones(30), tol=1e-14, max_iter=3)
    assert len(err.value.residuals) == 3


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock", "case1_mini"])
def test_oracle_s2_matches_reference(name):
    """The oracle's Method S2 (deterministic MFB) against the reference's own
    S2 sweep (tests/golden/make_golden_s2.py)."""
    from oracle import s3_cpu
    z = golden(name + "_s2")
    _, problem, grid, _ = case_from_golden(name)
    r = s3_cpu.run_s2(problem, grid, tol=TOL)
    assert _rel(np.array(r["lambdas"]), z["s2_lambda"]) <= 1e-9
    for key, (m, v) in r["moments"].items():
        mg, vg = z[f"mean__{key}"], z[f"var__{key}"]
        assert _rel(m, mg) <= 1e-8 or np.max(np.abs(m - mg)) <= 1e-12, key
        scale = max(float(np.max(mg ** 2)), 1e-300)
        assert (_rel(v, vg) <= max(1e-8, 10 * float(z[f"floor_var__{key}"]))
                or np.max(np.abs(v - vg)) / scale <= 1e-12), key


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock"])
def test_oracle_s1_matches_reference(name):
    """The oracle's Method S1 (matrix-free: a star solve per subdomain per
    CG iteration) against the reference's own S1 sweep
    (tests/golden/make_golden_s1.py)."""
    from oracle import s3_cpu
    z = golden(name + "_s1")
    _, problem, grid, _ = case_from_golden(name)
    r = s3_cpu.run_s1(problem, grid, tol=TOL)
    assert _rel(np.array(r["lambdas"]), z["s1_lambda"]) <= 1e-9
    assert abs(np.mean(r["iters"]) - np.mean(z["s1_iters"])) <= 0.05 * np.mean(z["s1_iters"]) + 1
    for key, (m, v) in r["moments"].items():
        mg, vg = z[f"mean__{key}"], z[f"var__{key}"]
        assert _rel(m, mg) <= 1e-8 or np.max(np.abs(m - mg)) <= 1e-12, key
        scale = max(float(np.max(mg ** 2)), 1e-300)
        assert _rel(v, vg) <= 1e-8 or np.max(np.abs(v - vg)) / scale <= 1e-12, key
