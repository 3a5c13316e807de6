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
        nt4 = (ndof[s] + 3) // 4
        w = 32 * (nt4 + (nt4 & 1))       # an even number of fragments per strip
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


def test_cg_point_order_chunks():
    """Sweep order of the multi-point CG: a permutation, longest points first,
    chunks of <= 8 that never split a reflection family of <= 8, single-point
    chunks in the tail, and fewer distinct local realizations per chunk than
    the plain longest-first order."""
    from paper_1802_06263_b200.adapter import load_config
    from paper_1802_06263_b200.interface import cg_point_order
    _, grid, _ = load_config(os.path.join(ROOT, "configs", "cfg4.json"))
    sub = np.arange(0, grid.n_real, 4)
    pts = np.asarray(grid.points)[sub]
    li = np.stack([np.asarray(l)[sub] for l in grid.local_indices])
    order, cptr = cg_point_order(pts, li, grid.local_points, tail=1184)
    n = len(sub)
    assert sorted(order.tolist()) == list(range(n))
    assert cptr[0] == 0 and cptr[-1] == n
    sizes = np.diff(cptr)
    assert sizes.min() >= 1 and sizes.max() <= 8
    assert np.all(sizes[np.searchsorted(cptr, n - 1184, side="left"):] == 1)
    key = np.abs(pts).max(axis=1)[order]
    assert np.all(np.diff(key) <= 1e-12)          # longest first

    def mult(o, bounds):
        tot = w = 0
        for a, b in zip(bounds[:-1], bounds[1:]):
            if b - a > 1:
                tot += sum(len(np.unique(li[r, o[a:b]])) for r in range(li.shape[0]))
                w += (b - a) * li.shape[0] / 8.0
        return tot / w
    plain = np.argsort(-np.abs(pts).max(axis=1), kind="stable")
    m_new = mult(order, cptr[:np.searchsorted(cptr, n - 1184) + 1])
    m_old = mult(plain, np.arange(0, n - 1184, 8))
    assert m_new < 0.9 * m_old, (m_new, m_old)
    # a small grid without structure still gets a valid order
    o2, c2 = cg_point_order(pts[:5], li[:, :5], grid.local_points, tail=0)
    assert sorted(o2.tolist()) == list(range(5)) and c2[-1] == 5


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_cg_stream_tasks_cover_every_row_once(name):
    """Tasks of the streamed multi-point CG: every mortar dof in exactly one
    task, 16-row tasks only where both subdomains' rows continue, their
    strips interleaved (second strip 64 doubles after the first, both
    flagged), every warp's 16-row tasks first, balanced shares."""
    from paper_1802_06263_b200.adapter import load_config
    from paper_1802_06263_b200.interface import cg_stream_tasks, cg_tasks
    problem, _, _ = load_config(os.path.join(ROOT, "configs", f"{name}.json"))
    n_sub, ndof, dof_ptr, dof_map = _maps(problem)
    nl = problem.space.n_dof
    tasks, sides, strips, pk_size = cg_tasks(n_sub, ndof, dof_ptr, dof_map, nl)
    lay = problem.layout
    region = np.array([lay.blocks[s].kl_region if lay.physics(s) == "darcy" else -1
                       for s in range(n_sub)])
    tab_s, strips_s = cg_stream_tasks(tasks, sides, strips, ndof, region)
    assert len(tab_s) % 16 == 0
    cov = np.zeros(nl, dtype=int)
    off = {(int(s), int(r0)): (int(o), int(f)) for s, r0, f, o in strips_s}
    for d0, so_i, so_j, w in tab_s:
        if w < 0:
            continue
        i, j, R = w & 0xfff, ((w >> 12) & 0xfff) - 1, w >> 24
        assert 1 <= R <= 16
        cov[d0:d0 + R] += 1
        for q in range(R):
            si, ai, sj, aj = sides[d0 + q]
            assert si == i and sj == j and ai == sides[d0, 1] + q
            assert j < 0 or aj == sides[d0, 3] + q
        for s_, a, so in ((i, sides[d0, 1], so_i), (j, sides[d0, 3], so_j)):
            if s_ < 0:
                continue
            o0, f0 = off[(s_, int(a))]
            assert o0 == so and (f0 >> 8) == (1 if R > 8 else 0)
            if R > 8:
                o1, f1 = off[(s_, int(a) + 8)]
                assert o1 == o0 + 64 and (f1 >> 8) == 1 and (f1 & 0xff) == R - 8
    assert np.all(cov == 1)
    for w in range(16):
        rows = [int(m) >> 24 for m in tab_s[w::16, 3] if m >= 0]
        assert rows == sorted(rows, key=lambda r: r <= 8)     # 16-row tasks first
    if name == "cfg4":
        assert sum(int(m) >> 24 > 8 for m in tab_s[:, 3] if m >= 0) == 108
