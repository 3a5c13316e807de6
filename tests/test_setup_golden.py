"""Host setup vs the golden fixtures: bit-exact grids and index maps.

The drop-in consumes the caller's sdmortar objects (adapter.py), so the
collocation nodes/weights, per-region local-index tables, interface list and
mortar dof maps ARE the reference's. This pins that the sdmortar + scipy of
the running environment (here, and the GPU box's baseline/_ref install)
reproduce, bit for bit, the setup the golden fixtures were generated with
(BASELINE.json north_star: grids and index maps bit-exact); the device
tables derived from them are pinned by test_adapter.py.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import ROOT, case_from_config, case_from_golden, golden

CASES = ["cfg1", "cfg2", "cfg3", "cfg5", "case1_mini", "darcy_twoblock"]


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _pins(problem, grid):
    lay = problem.layout
    ifaces = np.array([[g.index, g.i, g.j, "sd dd ss".split().index(g.kind),
                        0 if g.axis == "x" else 1, g.normal_sign] for g in lay.interfaces])
    dofs = [problem.space.sub_dofs(lay, s) for s in range(lay.n_subdomains)]
    return ifaces, np.concatenate(dofs), np.cumsum([0] + [len(d) for d in dofs])


@pytest.mark.parametrize("name", CASES)
def test_collocation_and_index_maps_bit_exact(name):
    z = golden(name)
    _, problem, grid, _ = case_from_golden(name)
    assert grid.n_real == int(z["n_real"])
    assert problem.space.n_dof == int(z["n_lambda"])
    assert list(grid.local_counts) == list(z["local_counts"])
    assert grid.points.tobytes() == z["grid_points"].tobytes()
    assert grid.weights.tobytes() == z["grid_weights"].tobytes()
    assert np.array_equal(np.stack(grid.local_indices), z["grid_local"])
    ifaces, dofs, ptr = _pins(problem, grid)
    assert np.array_equal(ifaces, z["ifaces"])
    assert np.array_equal(dofs, z["sub_dofs"])
    assert np.array_equal(ptr, z["sub_dofs_ptr"])


def test_cfg4_grid_hashes_bit_exact():
    """cfg4: 54,273-point level-3 Smolyak grid in 32 dims (hashes only)."""
    z = golden("cfg4")
    _, problem, grid, _ = case_from_config(f"{ROOT}/configs/cfg4.json")
    assert grid.n_real == int(z["n_real"]) == 54273
    assert list(grid.local_counts) == list(z["local_counts"])
    assert _sha(grid.points) == str(z["sha_points"])
    assert _sha(grid.weights) == str(z["sha_weights"])
    assert _sha(np.stack(grid.local_indices)) == str(z["sha_local"])
    ifaces, dofs, ptr = _pins(problem, grid)
    assert np.array_equal(dofs, z["sub_dofs"])
    assert problem.space.n_dof == 2720


def test_case1_sizes():
    """Sizes the reference pins for case1_mini (test_config.py:248-258)."""
    _, problem, grid, _ = case_from_golden("case1_mini")
    lay = problem.layout
    assert problem.space.n_dof == 48
    assert [len(problem.space.sub_dofs(lay, s)) for s in range(6)] == [12, 12, 20, 20, 16, 16]
    assert list(grid.local_counts) == [4, 8]
