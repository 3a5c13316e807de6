"""The streamed multi-point CG (mfb_cg_multi with pass lists, 16-row tasks, r
in tensor memory, chunked claims) against its own simpler forms on a cfg4
slice: scheduling must not change a bit, the streamed S p must agree with
the task loop to roundoff (interface.py:107-139, 238-247 per point)."""
import numpy as np
import pytest

from conftest import ROOT, case_from_config

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg4_slice(gpu):
    from sdmortar.collocation import CollocationGrid
    from paper_1802_06263_b200.interface import SweepEngine, get_plan
    _, problem, grid, _ = case_from_config(f"{ROOT}/configs/cfg4.json")
    pts = np.arange(0, grid.n_real, 23)[:2360]
    sub = CollocationGrid(grid.kind, grid.points[pts], grid.weights[pts], grid.splits,
                          [li[pts] for li in grid.local_indices],
                          list(grid.local_counts), list(grid.local_points))
    plan = get_plan(problem, sub)
    eng = SweepEngine(plan, keep_fields=False)
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    return eng, len(pts)


def _solve(eng, n, iters=300):
    # a fixed iteration budget: every point ends in MAX_ITER after `iters` steps
    lam, it, st, hist, _ = eng.solve_points(1e-30, iters, k0=0, n_pts=n, hist_cap=iters,
                                            kernel="multi")
    assert np.all(it.cpu().numpy() == iters)
    return lam


def test_claim_order_does_not_change_a_bit(cfg4_slice, monkeypatch):
    """Reflection-family order + chunked claims vs one point per claim in
    the plain longest-first order: same lambda bits, and reruns are equal."""
    from paper_1802_06263_b200 import interface
    eng, n = cfg4_slice
    a = _solve(eng, n)
    b = _solve(eng, n)
    monkeypatch.setattr(interface, "MULTI_CHUNKS", False)
    c = _solve(eng, n)
    import torch
    assert torch.equal(a, b)
    assert torch.equal(a, c)


def test_streamed_s_p_matches_task_loop(cfg4_slice, monkeypatch):
    """Pass lists with 16-row tasks vs the task loop: the same MMA sequence
    per (slot, row); only p . S p is added in another order. Compared after 5
    iterations: unpreconditioned CG at this conditioning (13k-74k iterations
    for n = 2,720) amplifies that roundoff by ~6x per early iteration
    (measured: 4e-16 after 1 iteration, 1.2e-15 after 5, 9e-4 after 20, 7e-3
    after 300), and the converged solutions agree again to 7e-13
    (tools/prof_cg_multi.py ... abs)."""
    from paper_1802_06263_b200 import interface
    eng, n = cfg4_slice
    assert eng.st._multi["list_cap"] > 0            # cfg4 runs the streamed kernel
    a = _solve(eng, n, iters=5)
    assert "streamed" in eng.cg_kernel_name
    monkeypatch.setattr(interface, "MULTI_STREAM", False)
    b = _solve(eng, n, iters=5)
    assert "streamed" not in eng.cg_kernel_name
    rel = float((a - b).abs().max() / b.abs().max())
    assert rel <= 1e-12, rel


def test_converged_lambda_solves_the_interface_system(cfg4_slice):
    """Size-independent check at cfg4's full interface size (n_lambda = 2,720,
    128 subdomains): for points solved to tol 1e-11 by the streamed kernel,
    the TRUE residual g - S lambda, with S applied on the host in the
    reference's own form (basis_apply, interface.py:238-247: ascending-sid
    scatter of B_i lambda|_i) from the plain block pool, is small. Nothing of
    the kernel's fragment strips, swizzled p, pass lists or tensor memory is
    shared with this check."""
    eng, n = cfg4_slice
    plan, st = eng.plan, eng.st
    pts = 16
    lam, it, status, hist, g = eng.solve_points(1e-11, 200000, k0=0, n_pts=pts, keep_g=True,
                                                kernel="multi")
    assert "streamed" in eng.cg_kernel_name
    assert np.all(status.cpu().numpy() == 0)
    blocks = st.blocks.cpu().numpy()
    local = np.asarray(plan.host.local)[:, :pts]
    L, G = lam.cpu().numpy(), g.cpu().numpy()
    worst = 0.0
    for k in range(pts):
        s_lam = np.zeros(plan.n_lambda)
        for i in range(plan.n_sub):
            nd = int(plan.ndof[i])
            dofs = plan.dof_map[plan.dof_ptr[i]:plan.dof_ptr[i + 1]]
            loc = int(local[plan.region[i], k]) if plan.region[i] >= 0 else 0
            off = int(st.blk_base[i]) + loc * nd * nd
            Bt = blocks[off:off + nd * nd].reshape(nd, nd)      # Bt[c, r] = B[r, c]
            s_lam[dofs] += Bt.T @ L[k, dofs]
        worst = max(worst, float(np.linalg.norm(G[k] - s_lam) / np.linalg.norm(G[k])))
    print(f"worst true relative residual over {pts} cfg4 points: {worst:.2e}")
    # the recursive residual is <= 1e-11; measured true residual 9.9e-12
    assert worst <= 1e-10, worst


def test_segmented_histories_reach_the_host_by_both_paths(gpu, monkeypatch):
    """SegmentedHist.to_host: small results land in pinned memory in one
    copy, large ones in a pageable array through a pinned staging buffer;
    the two paths return the same histories."""
    from conftest import case_from_golden
    from paper_1802_06263_b200 import interface
    from paper_1802_06263_b200.interface import SweepEngine, get_plan
    _, problem, grid, _ = case_from_golden("cfg2")
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, keep_fields=False)
    eng.kl_fields()
    eng.build_bases()
    lam, iters, status, hist, _ = eng.solve_points(1e-11, 10 * plan.n_lambda, kernel="multi")
    it = iters.cpu().numpy().astype(np.int64)
    a = hist.to_host(it)
    monkeypatch.setattr(interface, "PINNED_HIST_BYTES_MAX", 0)
    monkeypatch.setattr(interface, "_HIST_STAGE_DOUBLES", 1000)      # several chunks
    b = hist.to_host(it)
    assert len(a) == len(b) == grid.n_real
    for k in (0, grid.n_real // 2, grid.n_real - 1):
        assert np.array_equal(a.array(k), b.array(k)) and len(a.array(k)) == it[k]
    assert a.array(0)[-1] <= 1e-11


def test_basis_blocks_are_exactly_symmetric(gpu):
    """Every flux-basis block the S3 sweep stores is exactly symmetric: the
    Darcy condensation's by construction, the banded LU's after
    mfb_blocks_symmetrize (the reference's SuperLU blocks: symmetric to 3e-13,
    SURVEY 8a a6). The unpreconditioned CG pays ~10% more iterations for 1e-12
    of asymmetry (profiles/r02/cg_iterations_vs_reference.txt)."""
    import torch
    from conftest import case_from_golden
    from paper_1802_06263_b200.interface import SweepEngine, get_plan
    _, problem, grid, _ = case_from_golden("cfg2")
    plan = get_plan(problem, grid)
    eng = SweepEngine(plan, keep_fields=False)
    eng.kl_fields()
    eng.build_bases()
    eng.check_info()
    st = eng.st
    for s in range(plan.n_sub):
        nd, nloc, off = int(plan.ndof[s]), int(st.n_loc[s]), int(st.blk_base[s])
        B = st.blocks[off:off + nloc * nd * nd].view(nloc, nd, nd)
        assert torch.equal(B, B.transpose(1, 2)), s
