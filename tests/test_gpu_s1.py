"""Solves with stored factors (mfb_systems_apply, the star solves of Method
S1): applied to unit mortar coefficients they must reproduce the
factorization's own solution columns X = S^-1 Q and the flux-basis columns
B = Q^T X, for Darcy (generic band path) and Stokes systems, with and
without the rigid-body kernel projection."""

import ctypes

import numpy as np
import pytest

from conftest import case_from_golden

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["cfg1", "case1_mini", "cfg2"])
def test_apply_with_stored_factors_reproduces_the_solves(gpu, name):
    import torch
    from paper_1802_06263_b200 import _lib
    from paper_1802_06263_b200.interface import SweepEngine, get_plan
    from paper_1802_06263_b200.plan import _ptr
    _, problem, grid, _ = case_from_golden(name)
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, method="S2", darcy_kernel="band", keep_factors=True)
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    st = eng.st
    L = _lib.lib()
    Xall = st.X.cpu().numpy()
    blocks = st.blocks.cpu().numpy()
    checked = set()
    for w in st.waves:
        idx = w["idx"]
        xoff = w["xoff"].cpu().numpy()
        pat = w["pat"].cpu().numpy()
        # a few systems of every subdomain (all columns of each)
        pick = [j for j, g in enumerate(idx) if st.systems[g][1] < 2]
        items, cols = [], []
        for j in pick:
            nd = int(plan.ndof[pat[j]])
            for c in range(nd):
                items.append(j)
                cols.append(c)
        nd_max = int(plan.ndof.max())
        V = np.zeros((len(items), nd_max))
        V[np.arange(len(items)), cols] = 1.0
        n_max = max(int(plan.patterns[pat[j]].n + plan.patterns[pat[j]].nb) for j in pick)
        dV = torch.as_tensor(V, device="cuda")
        dX = torch.zeros((len(items), n_max), dtype=torch.float64, device="cuda")
        dR = torch.zeros((len(items), nd_max), dtype=torch.float64, device="cuda")
        d_items = torch.as_tensor(np.array(items, dtype=np.int32), device="cuda")
        _lib.check(L.mfb_systems_apply(
            _ptr(plan.pat_dev), len(items), _ptr(d_items), _ptr(w["pat"]), _ptr(st.work),
            _ptr(w["woff"]), _ptr(dV), nd_max, _ptr(dX), n_max, _ptr(dR), nd_max, n_max,
            ctypes.c_void_p(eng.stream.cuda_stream)), "mfb_systems_apply")
        X = dX.cpu().numpy()
        R = dR.cpu().numpy()
        for t, (j, c) in enumerate(zip(items, cols)):
            P = plan.patterns[pat[j]]
            nd, nn = int(P.ndof), int(P.n + P.nb)
            ref = Xall[xoff[j]: xoff[j] + nn * (nd + 1)].reshape(nn, nd + 1)[:, c]
            # roundoff of a different summation order than the blocked rhs path
            assert np.max(np.abs(X[t, :nn] - ref)) <= 1e-9 * max(np.max(np.abs(ref)), 1e-300)
            g = idx[j]
            Bt = blocks[st.sys_boff[g]: st.sys_boff[g] + nd * nd].reshape(nd, nd)
            bcol = Bt[c]                               # column c of B
            assert np.max(np.abs(R[t, :nd] - bcol)) <= 1e-10 * np.max(np.abs(Bt))
            checked.add((int(pat[j]), int(P.nb) > 0))
    assert any(nbpos for _, nbpos in checked) or name != "cfg2"
