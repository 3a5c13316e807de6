"""The reference's run writers (sdmortar/output.py: VTK, moments.csv,
stats.csv, manifest.json -- SURVEY 8f row 3) accept this package's problem,
grid and RunResult unchanged, and write the same bytes as for the
reference's own objects holding the same numbers.

CPU only; needs the read-only reference mount (skipped elsewhere, e.g. on
the GPU box). The moments are the reference's own (golden fixture), so the
comparison isolates the host objects and the result/stats containers."""

import filecmp
import json
import os
import sys

import numpy as np
import pytest

from conftest import case_from_golden, golden

REF = "/root/reference/pkg/src"


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock"])
def test_reference_writers_accept_our_objects(name, tmp_path):
    if not os.path.isdir(REF):
        pytest.skip("reference package not mounted")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    from sdmortar import interface as ref_iface
    from sdmortar.config import build_from_config as ref_build
    from sdmortar.config import validate_config as ref_validate
    from sdmortar.output import write_outputs

    from paper_1802_06263_b200.interface import RunResult, SolveStats

    z = golden(name)
    cfg, problem, grid, _ = case_from_golden(name)
    raw = json.loads(str(z["config_json"]))
    ref_cfg = ref_validate(raw)
    ref_problem, ref_grid, _ = ref_build(ref_cfg)
    keys = [k[len("mean__"):] for k in z.files if k.startswith("mean__")]
    moments = {k: (z[f"mean__{k}"], z[f"var__{k}"]) for k in keys}
    n_sub = problem.layout.n_subdomains
    iters = [int(x) for x in z["s3_iters"]]

    ours = SolveStats.new("S3", n_sub)
    ours.factorizations[:] = z["stats_factorizations"]
    ours.backsolves[:] = z["stats_backsolves"]
    ours.basis_backsolves[:] = z["stats_basis_backsolves"]
    ours.cg_iters = iters
    ours.n_real = grid.n_real
    theirs = ref_iface.SolveStats.new("S3", n_sub)
    theirs.factorizations[:] = z["stats_factorizations"]
    theirs.backsolves[:] = z["stats_backsolves"]
    theirs.basis_backsolves[:] = z["stats_basis_backsolves"]
    theirs.cg_iters = iters
    theirs.n_real = ref_grid.n_real

    lam = list(z["s3_lambda"])
    res_ours = RunResult(moments, ours, lam, [[] for _ in lam], grid)
    res_ref = ref_iface.RunResult(moments, theirs, lam, [[] for _ in lam], ref_grid)
    p1 = write_outputs(str(tmp_path / "ours"), cfg, problem, grid, res_ours)
    p2 = write_outputs(str(tmp_path / "ref"), ref_cfg, ref_problem, ref_grid, res_ref)
    files = p1["vtk"] + [p1["moments_csv"], p1["stats_csv"], p1["manifest"]]
    refs = p2["vtk"] + [p2["moments_csv"], p2["stats_csv"], p2["manifest"]]
    for a, b in zip(files, refs):
        assert filecmp.cmp(a, b, shallow=False), (os.path.basename(a), name)
    assert np.array_equal(np.loadtxt(p1["stats_csv"], delimiter=",", skiprows=1,
                                     usecols=(2, 3, 4)),
                          np.loadtxt(p2["stats_csv"], delimiter=",", skiprows=1,
                                     usecols=(2, 3, 4)))
