"""The drop-in consumes the reference's own objects (adapter.py).

* the device tables built from `sdmortar.config.build_from_config` objects are
  byte-identical to the tables of round 1's host setup (fixture written by
  tools/host_table_hashes.py before that setup was deleted);
* the error classes ARE sdmortar.errors' classes;
* the plan cache notices in-place edits of the caller's mutable problem.
"""

import json
import os

import pytest

from conftest import ROOT

FIX = os.path.join(ROOT, "tests", "golden", "host_tables_sha.json")


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "case1_mini",
                                  "darcy_twoblock"])
def test_tables_from_sdmortar_objects_byte_identical(name):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    from host_table_hashes import raw_config, table_hashes
    from sdmortar.config import build_from_config, validate_config
    with open(FIX) as fh:
        want = json.load(fh)[name]
    problem, grid, _ = build_from_config(validate_config(raw_config(name)))
    assert type(problem).__module__ == "sdmortar.problem"
    assert type(grid).__module__ == "sdmortar.collocation"
    got = table_hashes(problem, grid)
    assert sorted(got) == sorted(want)
    bad = [k for k in want if got[k] != want[k]]
    assert not bad, bad[:10]


def test_error_classes_are_the_reference_classes():
    import sdmortar.errors as ref
    from paper_1802_06263_b200 import errors
    for name in ("ConfigError", "ConvergenceError", "SingularOperatorError", "SizeCapError"):
        assert getattr(errors, name) is getattr(ref, name)
    e = errors.ConvergenceError("x", [1.0, 0.5])
    assert isinstance(e, ref.ConvergenceError) and e.residuals == [1.0, 0.5]


def test_plan_fingerprint_sees_in_place_edits():
    from conftest import case_from_golden
    from paper_1802_06263_b200.interface import _plan_fingerprint
    from sdmortar.darcy import DarcyBC
    _, problem, grid, _ = case_from_golden("cfg1")
    f0 = _plan_fingerprint(problem, grid)
    assert _plan_fingerprint(problem, grid) == f0
    sid = next(s for s in range(problem.layout.n_subdomains)
               if problem.layout.physics(s) == "darcy")
    problem.bcs.setdefault(sid, {})["bottom"] = DarcyBC("pressure", lambda x, y: 1.0 + 0 * x)
    f1 = _plan_fingerprint(problem, grid)
    assert f1 != f0
    grid.weights[0] += 1.0
    assert _plan_fingerprint(problem, grid) != f1
