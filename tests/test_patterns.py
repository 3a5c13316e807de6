"""Host-side system patterns (discretization.py) reproduce the reference blocks.

A dense CPU evaluation of each subdomain's parametrised pattern (the matrix
the device assembles) is solved with numpy and read out exactly like the
device `extract` kernel; the resulting flux-basis blocks must match the
reference's `compute_flux_basis` (golden fixtures) -- this checks the
band numbering, the mortar columns Q, the border (rigid-body) treatment and
the readout signs independently of the GPU.
"""

import numpy as np
import pytest

import pattern_emu
from paper_1802_06263_b200.adapter import darcy_sids
from conftest import case_from_golden, golden


def _k0(problem, grid):
    from oracle import s3_cpu
    off, cur = {}, 0
    for s in darcy_sids(problem):
        off[s] = cur
        cur += problem.meshes[s].n_cells
    K0 = np.zeros(cur)
    zero = np.zeros(grid.n_dims)
    for s in darcy_sids(problem):
        K0[off[s]:off[s] + problem.meshes[s].n_cells] = s3_cpu.realize(problem, s, zero)
    return off, K0


@pytest.mark.parametrize("name", ["cfg1", "case1_mini", "darcy_twoblock"])
def test_pattern_blocks_match_reference(name):
    from oracle import s3_cpu
    from paper_1802_06263_b200.discretization import darcy_pattern, stokes_pattern
    z = golden(name)
    _, problem, grid, _ = case_from_golden(name)
    off, K0 = _k0(problem, grid)
    plan = s3_cpu.s3_plan(problem, grid)
    for s in range(problem.layout.n_subdomains):
        if problem.layout.physics(s) == "darcy":
            pat = darcy_pattern(problem, s)
            for loc in (0, len(plan[s]) - 1):
                r = pattern_emu.solve(pat, s3_cpu.realize(problem, s, plan[s][loc]))
                Bg = z[f"B__{s}__{loc}"]
                assert np.max(np.abs(r["B"] - Bg)) <= 1e-12 * np.max(np.abs(Bg))
                assert np.max(np.abs(r["B"] - r["B"].T)) <= 1e-12 * np.max(np.abs(Bg))
        else:
            pat = stokes_pattern(problem, s, off, K0)
            r = pattern_emu.solve(pat, K0)
            Bg = z[f"B__{s}__0"]
            assert np.max(np.abs(r["B"] - Bg)) <= 1e-10 * np.max(np.abs(Bg))


def test_pattern_bar_and_fields_match_oracle():
    """Bar jump h and postprocessed star/bar fields vs the oracle's solves."""
    from oracle import s3_cpu
    from paper_1802_06263_b200.discretization import darcy_pattern, stokes_pattern
    _, problem, grid, _ = case_from_golden("cfg1")
    off, K0 = _k0(problem, grid)
    plan = s3_cpu.s3_plan(problem, grid)
    for s in range(problem.layout.n_subdomains):
        darcy = problem.layout.physics(s) == "darcy"
        K = s3_cpu.realize(problem, s, plan[s][0]) if darcy else K0
        pat = darcy_pattern(problem, s) if darcy else stokes_pattern(problem, s, off, K0)
        r = pattern_emu.solve(pat, K)
        Kf = {s: K} if darcy else s3_cpu.mean_field_K(problem, grid.n_dims)
        op = s3_cpu.assemble(problem, s, Kf)
        dofs, maps = s3_cpu.local_positions(problem, s)
        u, p = s3_cpu.bar_solve(op)
        h = s3_cpu.restrict(s3_cpu.side_values(problem, s, op, u), maps, len(dofs))
        assert np.max(np.abs(r["h"] - h)) <= 1e-10 * max(np.max(np.abs(h)), 1e-30)
        fb = op.postprocess(u, p)
        flat = np.concatenate([np.ravel(fb[k]) for k in ("u", "p", "cv", "cp")])
        assert np.max(np.abs(r["Fb"] - flat)) <= 1e-10 * max(np.max(np.abs(flat)), 1e-30)
        lam = np.zeros(problem.space.n_dof)
        lam[dofs[0]] = 1.0
        us, ps = s3_cpu.star_solve(problem, s, op, lam)
        fs = op.postprocess(us, ps)
        flat = np.concatenate([np.ravel(fs[k]) for k in ("u", "p", "cv", "cp")])
        # star fields of unit mortar dof 0 are -M[:, 0]
        assert np.max(np.abs(-r["M"][:, 0] - flat)) <= 1e-10 * max(np.max(np.abs(flat)), 1e-30)
