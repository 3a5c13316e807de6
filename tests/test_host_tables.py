"""Host-side tables of the device path (CPU only): the multi-point CG's work
items and packed-strip layout (interface.cg_tasks) and the packed residual
histories (interface.ResidualHistories)."""

import os

import numpy as np
import pytest

from conftest import ROOT, case_from_golden


def _maps(problem):
    lay = problem.layout
    dofs = [problem.space.sub_dofs(lay, s) for s in range(lay.n_subdomains)]
    ndof = np.array([len(d) for d in dofs])
    return lay.n_subdomains, ndof, np.cumsum([0] + list(ndof)), np.concatenate(dofs)


@pytest.mark.parametrize("name", ["cfg1", "darcy_twoblock", "case1_mini", "cfg2", "cfg4"])
def test_cg_tasks_cover_every_row_once(name):
    from paper_1802_06263_b200.adapter import load_config
    from paper_1802_06263_b200.interface import cg_tasks
    if name in ("cfg2", "cfg4"):
        problem, _, _ = load_config(os.path.join(ROOT, "configs", f"{name}.json"))
    else:
        _, problem, _, _ = case_from_golden(name)
    n_sub, ndof, dof_ptr, dof_map = _maps(problem)
    nl = problem.space.n_dof
    tasks, sides, strips, pk_size = cg_tasks(n_sub, ndof, dof_ptr, dof_map, nl)
    # every mortar dof in exactly one task; a task's dofs share both sides
    # and have consecutive rows in both subdomains
    cov = np.zeros(nl, dtype=int)
    for d0, so_i, so_j, w in tasks:
        i, j, R = w & 0xfff, ((w >> 12) & 0xfff) - 1, w >> 24
        assert 1 <= R <= 8
        cov[d0:d0 + R] += 1
        for q in range(R):
            si, ai, sj, aj = sides[d0 + q]
            assert si == i and sj == j
            assert ai == sides[d0, 1] + q
            if j >= 0:
                assert aj == sides[d0, 3] + q
    assert np.all(cov == 1)
    # sides: the stacked rows of each dof, lower subdomain first
    for d in range(nl):
        i, ai, j, aj = sides[d]
        assert dof_map[dof_ptr[i] + ai] == d
        if j >= 0:
            assert i < j and dof_map[dof_ptr[j] + aj] == d
    # strips partition every block's rows; offsets are whole fragment runs
    for s in range(n_sub):
        mine = strips[strips[:, 0] == s]
        w = 32 * ((ndof[s] + 3) // 4)
        rows = np.zeros(ndof[s], dtype=int)
        for _, r0, R, off in mine:
            rows[r0:r0 + R] += 1
            assert off % w == 0 and off < pk_size[s]
        assert np.all(rows == 1)
        assert pk_size[s] == w * len(mine)
    # tasks are ordered most expensive first (warps take them round robin)
    cost = [ndof[w & 0xfff] + (ndof[((w >> 12) & 0xfff) - 1] if (w >> 12) & 0xfff else 0)
            for w in tasks[:, 3]]
    assert all(a >= b for a, b in zip(cost, cost[1:]))


def test_residual_histories_behave_like_lists():
    from paper_1802_06263_b200.interface import ResidualHistories
    iters = [3, 0, 2]
    flat = np.array([0.5, 0.25, 1e-12, 0.75, 1e-13])
    h = ResidualHistories(flat, iters)
    assert len(h) == 3
    assert h[0] == [0.5, 0.25, 1e-12] and h[1] == [] and h[2] == [0.75, 1e-13]
    assert h[-1] == h[2] and h[0:2] == [h[0], h[1]]
    assert [len(x) for x in h] == iters
    assert np.shares_memory(h.array(2), flat)
    with pytest.raises(IndexError):
        h[3]


def test_residual_histories_from_the_padded_device_array():
    """run_method keeps the [points, cap] history array the device wrote
    (no host repacking on the end-to-end path); rows, views and the lazily
    built flat storage behave as the flat-built histories."""
    from paper_1802_06263_b200.interface import ResidualHistories
    pad = np.array([[0.5, 0.25, 1e-12, 9.0], [9.0] * 4, [0.75, 1e-13, 9.0, 9.0]])
    h = ResidualHistories.from_padded(pad, [3, 0, 2])
    ref = ResidualHistories(np.array([0.5, 0.25, 1e-12, 0.75, 1e-13]), [3, 0, 2])
    assert len(h) == 3 and [h[k] for k in range(3)] == [ref[k] for k in range(3)]
    assert h[-1] == ref[-1] and h[0:2] == ref[0:2]
    assert np.shares_memory(h.array(2), pad)
    assert np.array_equal(h.flat, ref.flat) and np.array_equal(h.offsets, ref.offsets)
    with pytest.raises(IndexError):
        h[3]
