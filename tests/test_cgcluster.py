"""Host tables of the cluster CG (paper_1802_06263_b200/cgcluster.py), CPU only:
the per-rank partition, ownership, halo peers, cut rows and tasks, emulated
on the host, must reproduce the interface operator S p = sum_i R_i^T B_i R_i p
(basis_apply, reference interface.py:238-247) for every cluster shape."""

import os

import numpy as np
import pytest

from conftest import ROOT, case_from_golden


def _setup(name):
    from paper_1802_06263_b200.adapter import load_config
    if name in ("cfg2", "cfg4"):
        problem, _, _ = load_config(os.path.join(ROOT, "configs", f"{name}.json"))
    else:
        _, problem, _, _ = case_from_golden(name)
    lay = problem.layout
    dofs = [np.asarray(problem.space.sub_dofs(lay, s)) for s in range(lay.n_subdomains)]
    ndof = np.array([len(d) for d in dofs])
    centers = np.array([[(b.rect[0] + b.rect[2]) / 2, (b.rect[1] + b.rect[3]) / 2]
                        for b in lay.blocks])
    region = np.array([b.kl_region if lay.physics(s) == "darcy" else -1
                       for s, b in enumerate(lay.blocks)])
    return problem, dofs, ndof, centers, region


@pytest.mark.parametrize("name,C,NP", [("cfg1", 2, 8), ("case1_mini", 2, 16), ("cfg2", 4, 16),
                                       ("cfg2", 8, 8), ("cfg4", 4, 16), ("cfg4", 8, 16),
                                       ("cfg4", 2, 8)])
def test_cluster_tables_emulate_apply(name, C, NP):
    from paper_1802_06263_b200.cgcluster import cluster_tables, emulate_apply
    from paper_1802_06263_b200.interface import cg_tasks
    problem, dofs, ndof, centers, region = _setup(name)
    n_sub, nl = len(dofs), problem.space.n_dof
    dof_ptr = np.cumsum([0] + list(ndof))
    dof_map = np.concatenate(dofs)
    tasks, sides, strips, pk_size = cg_tasks(n_sub, ndof, dof_ptr, dof_map, nl)
    pk_base = np.concatenate([[0], np.cumsum(pk_size.astype(np.int64))])[:-1]
    ct = cluster_tables(n_sub, ndof, dof_ptr, dof_map, nl, region, centers, C, NP,
                        tasks, sides, pk_base, pk_size)
    hdr = ct["hdr"]
    # every dof owned exactly once; owned rows are the first rows of p
    own_all = np.concatenate([ct["tab"][h[5]:h[5] + h[0]] for h in hdr])
    assert np.array_equal(np.sort(own_all), np.arange(nl))
    # units per rank reference only that rank's column maps and strips
    for h in hdr:
        units = ct["tab"][h[7]:h[7] + 8 * h[2]].reshape(-1, 8)
        for nd, reg, psz, cmo, ns, so, ps, _ in units:
            assert 0 <= cmo and cmo + nd <= h[4] and 0 <= so and so + ns <= h[10]
    rng = np.random.default_rng(7)
    blocks = []
    for s in range(n_sub):
        a = rng.standard_normal((ndof[s], ndof[s]))
        blocks.append(a + a.T)
    strip_at = {int(pk_base[s]) + int(off): (int(s), int(r0)) for s, r0, _, off in strips}
    P = rng.standard_normal((nl, NP))
    Sp = emulate_apply(ct, lambda s: blocks[s], lambda pk: strip_at[int(pk)], P)
    ref = np.zeros_like(P)
    for s in range(n_sub):
        ref[dofs[s]] += blocks[s] @ P[dofs[s]]
    assert np.allclose(Sp, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())


def test_partition_cfg4_is_column_strips():
    from paper_1802_06263_b200.cgcluster import partition
    problem, dofs, ndof, centers, _ = _setup("cfg4")
    part = partition(len(dofs), centers, ndof.astype(float) ** 2, 4)
    # 16 x 8 grid of subdomains, sid = row * 16 + column: four strips of 4 columns
    cols = np.arange(len(dofs)) % 16
    assert np.array_equal(part, cols // 4)


def test_residual_histories_from_segments():
    from paper_1802_06263_b200.interface import ResidualHistories
    seg = 4
    iters = np.array([0, 3, 4, 9])
    rng = np.random.default_rng(1)
    hist = [rng.standard_normal(n) for n in iters]
    tab = -np.ones((4, 3), dtype=np.int32)
    pool = np.full(16 * seg, np.nan)
    nxt = 0
    for k in (3, 1, 2):                   # segments drawn out of order
        for i in range(0, iters[k], seg):
            tab[k, i // seg] = nxt
            chunk = hist[k][i:i + seg]
            pool[nxt * seg:nxt * seg + len(chunk)] = chunk
            nxt += 1
    h = ResidualHistories.from_segments(pool, tab, iters, seg)
    for k in range(4):
        assert h[k] == hist[k].tolist()
    assert np.array_equal(h.flat, np.concatenate(hist))
    assert np.array_equal(h.offsets, np.concatenate([[0], np.cumsum(iters)]))
