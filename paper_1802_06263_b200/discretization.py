"""Subdomain systems as parametrised, banded patterns for the device solver.

Host setup (realization-independent). For every subdomain this module
builds the *structure* of the linear system the reference factors with
SuperLU -- the mixed RT0/P0 Darcy saddle matrix (reference darcy.py:64-147)
and the Taylor-Hood Stokes matrix with BJS friction and rigid-body kernel
constraints (reference stokes.py:109-298) -- but not its values: each
matrix entry is a short list of terms `c`, `c / K[k]` or `c / sqrt(K[k])`
that the device evaluates for the realization's permeability. The unknowns
are renumbered so the matrix is banded:

* Darcy: per cell row iy, [kept vertical edges, kept bottom edges, cells],
  then the kept top edges of the last row; half-bandwidth 3 nx + 1.
* Stokes: lattice-row order, (u_x, u_y[, p]) per P2 node; the Lagrange
  rows of the rigid-body kernel (dense) and k pinned velocity dofs that
  make the interior block regular go to a small dense border.

Right-hand sides are the mortar columns Q (one per local mortar dof; the
reference's star solve of unit mortar data, interface.py:218-235,
problem.py:114-130) and the bar column (darcy.py:178-193,
stokes.py:325-361). Readouts: B = Q^T X (interface.py:210-215 with
problem.py:132-148) and the postprocessed fields (problem.py:150-158).
"""

from dataclasses import dataclass, field

import numpy as np

from .adapter import (OUTWARD_SIGN, P2_EDGE_MASS, SIDES, DarcyBC, StokesBC, cell_edge_table,
                      edge_midpoint)

TERM_CONST, TERM_INV_K, TERM_INV_SQRT_K = 0, 1, 2

# Dunavant degree-4 triangle rule (stokes.py:28-35); weights sum to 1/2
_DUN_W = np.array([0.223381589678011] * 3 + [0.109951743655322] * 3) * 0.5
_DA, _DB = 0.445948490915965, 0.091576213509771
_DUN_P = np.array([[_DA, _DA], [1 - 2 * _DA, _DA], [_DA, 1 - 2 * _DA],
                   [_DB, _DB], [1 - 2 * _DB, _DB], [_DB, 1 - 2 * _DB]])
_GL3_X = np.array([-np.sqrt(3 / 5), 0.0, np.sqrt(3 / 5)])
_GL3_W = np.array([5, 8, 5]) / 9.0


@dataclass
class Pattern:
    """Host copy of one MfbPattern (see include/mfb.h)."""

    sid: int
    physics: str
    n: int
    kl: int
    ku: int
    nb: int
    ndof: int
    nfield: int
    e_row: np.ndarray
    e_col: np.ndarray
    e_tptr: np.ndarray
    t_kind: np.ndarray
    t_c: np.ndarray
    t_k: np.ndarray
    E: np.ndarray
    G: np.ndarray
    q_ptr: np.ndarray
    q_row: np.ndarray
    q_val: np.ndarray
    bar_const: np.ndarray
    b_row: np.ndarray
    b_tptr: np.ndarray
    bt_kind: np.ndarray
    bt_c: np.ndarray
    bt_k: np.ndarray
    h_lift: np.ndarray
    p_ptr: np.ndarray
    p_col: np.ndarray
    p_val: np.ndarray
    f_lift: np.ndarray
    field_layout: list = field(default_factory=list)  # [(name, start, shape)]
    kernel_dim: int = 0

    @property
    def ldab(self):
        return 2 * self.kl + self.ku + 1

    @property
    def work_doubles(self):
        # band, rhs rows, BAND_GROUP_MAX + 1 panel-publication slots ((kl + 16)
        # x 16 scaled factors + 32 scales + 16 doubles of pivots/flag), then n reciprocal U
        # diagonals, the inverses of the 16 x 16 diagonal U blocks, the n
        # panel pivot positions (ints) and the (kl + 16) x 16 multiplier
        # panels (mfb_band.cu)
        w = (self.ldab * self.n + self.n * (self.ndof + 1) + 1
             + 17 * ((self.kl + 16) * 16 + 48) + self.n + 256 * ((self.n + 15) // 16) + 1
             + (self.n + 1) // 2 + 1 + ((self.n + 15) // 16) * (self.kl + 16) * 16)
        return w + (w & 1)                 # even: every system's slots stay 16-byte aligned

    @property
    def x_doubles(self):
        return (self.n + self.nb) * (self.ndof + 1)

    @property
    def algorithmic_flops(self):
        """F = 2 n w^2 + 4 n w N_dof, w = half-bandwidth of the ordering."""
        w = max(self.kl, self.ku)
        return 2.0 * self.n * w * w + 4.0 * self.n * w * self.ndof

    @property
    def smem_doubles(self):
        # band_solve_kernel (NB = 16): panel (kl + 16) x 17, U12 + staging 2 x 16 x ust,
        # rhs rows 16 x (ndof + 1)
        # back substitution reuses it: window 8 x (kl + ku + 32), two U blocks
        # 16 x ldu, solved rows 16 x 8, two U11 blocks
        ust = (self.kl + self.ku + 16) | 1
        ldu = ((self.kl + self.ku + 15) & ~7) + 4
        lu = ((self.kl + 16) * 17 + 16 * ust + max(16 * ust, 3 * 8 * 160)
              + 16 * (self.ndof + 1))
        bs = 8 * (self.kl + self.ku + 32) + 2 * 16 * ldu + 16 * 8 + 2 * 16 * 16
        return max(lu, bs)


class _TermTable:
    """Accumulate (row, col) -> term list, then group into CSR-like arrays."""

    def __init__(self):
        self.rows, self.cols, self.kind, self.c, self.k = [], [], [], [], []

    def add(self, rows, cols, kind, c, k=None):
        rows = np.atleast_1d(np.asarray(rows, dtype=np.int64))
        cols = np.broadcast_to(np.asarray(cols, dtype=np.int64), rows.shape)
        self.rows.append(rows)
        self.cols.append(np.array(cols))
        self.kind.append(np.full(rows.shape, kind, dtype=np.int32))
        self.c.append(np.broadcast_to(np.asarray(c, dtype=float), rows.shape).copy())
        kk = np.zeros(rows.shape, dtype=np.int64) if k is None else \
            np.broadcast_to(np.asarray(k, dtype=np.int64), rows.shape)
        self.k.append(np.array(kk))

    def arrays(self):
        if not self.rows:
            z = np.zeros(0, dtype=np.int64)
            return z, z, z, z.astype(np.int32), np.zeros(0), z
        rows = np.concatenate(self.rows)
        cols = np.concatenate(self.cols)
        kind = np.concatenate(self.kind)
        c = np.concatenate(self.c)
        k = np.concatenate(self.k)
        # one stable sort on the combined (row, col) key == lexsort((cols, rows))
        key = (rows << 32) | cols
        order = np.argsort(key, kind="stable")    # stable: keeps insertion order
        rows, cols, kind, c, k = rows[order], cols[order], kind[order], c[order], k[order]
        new = np.ones(len(rows), dtype=bool)
        new[1:] = (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])
        starts = np.nonzero(new)[0]
        tptr = np.append(starts, len(rows))
        return rows[starts], cols[starts], tptr, kind, c, k

    def constant_dense_at(self, shape):
        """Sum constant terms into a dense matrix (for border blocks)."""
        out = np.zeros(shape)
        for r, cc, kd, v in zip(self.rows, self.cols, self.kind, self.c):
            if np.any(kd != TERM_CONST):
                raise ValueError("border entries must be realization independent")
            np.add.at(out, (r, cc), v)
        return out


def _csr(rows, cols, vals, n_rows):
    rows = np.asarray(rows, dtype=np.int64)
    order = np.argsort(rows, kind="stable")
    ptr = np.zeros(n_rows + 1, dtype=np.int64)
    np.add.at(ptr, rows + 1, 1)
    return (np.cumsum(ptr), np.asarray(cols, dtype=np.int64)[order],
            np.asarray(vals, dtype=float)[order])


def _local_mortar_positions(problem, sid):
    """{(iface, comp): local positions of its scalar functions} (interface.py:197-207)."""
    pos, start = {}, 0
    for g in problem.layout.interfaces_of(sid):
        b = problem.space.block(g.index)
        for c in range(b.n_comp):
            pos[(g.index, c)] = start + np.arange(b.n_scalar) * b.n_comp + c
        start += b.n_dof
    return pos, start


# ============================================================== Darcy =====
def darcy_pattern(problem, sid):
    mesh = problem.meshes[sid]
    nx, ny = mesh.nx, mesh.ny
    bcs = problem.bcs.get(sid, {})
    traces = problem.traces[sid]
    nu = problem.physics.nu_d
    iface_edges = set(int(e) for t in traces for e in t.edges)
    noflow, pressure = set(), {}
    for side in SIDES:
        bc = bcs.get(side, DarcyBC("noflow"))
        for e in mesh.boundary_edges(side):
            e = int(e)
            if e in iface_edges:
                continue
            if bc.kind == "noflow":
                noflow.add(e)
            elif bc.kind == "pressure":
                pressure[e] = (side, bc.value)
            else:
                raise ValueError(f"unknown darcy bc {bc.kind!r}")
    if not pressure and not iface_edges:
        from .errors import SingularOperatorError
        raise SingularOperatorError("darcy subdomain has no pressure data and no "
                                    "interface; pressure is undetermined")
    # band numbering
    edge_idx = -np.ones(mesh.n_edges, dtype=np.int64)
    cell_idx = np.empty(mesh.n_cells, dtype=np.int64)
    nxt = 0
    for iy in range(ny + 1):
        if iy < ny:
            for ix in range(nx + 1):
                e = mesh.vedge(ix, iy)
                if e not in noflow:
                    edge_idx[e] = nxt
                    nxt += 1
        for ix in range(nx):
            e = mesh.hedge(ix, iy)
            if e not in noflow:
                edge_idx[e] = nxt
                nxt += 1
        if iy < ny:
            for ix in range(nx):
                cell_idx[mesh.cell(ix, iy)] = nxt
                nxt += 1
    n = nxt
    E = cell_edge_table(mesh)                     # w e s n
    cells = np.arange(mesh.n_cells)
    area = mesh.hx * mesh.hy
    tt = _TermTable()
    # A = nu (K^-1 u, v): per cell 1/3 diagonal, 1/6 w-e and s-n (darcy.py:118-131)
    for a, b, m in ((0, 0, 1 / 3), (1, 1, 1 / 3), (0, 1, 1 / 6), (1, 0, 1 / 6),
                    (2, 2, 1 / 3), (3, 3, 1 / 3), (2, 3, 1 / 6), (3, 2, 1 / 6)):
        ra, rb = edge_idx[E[:, a]], edge_idx[E[:, b]]
        ok = (ra >= 0) & (rb >= 0)
        tt.add(ra[ok], rb[ok], TERM_INV_K, nu * area * m, cells[ok])
    # B = -(div v, w) and its transpose (darcy.py:132-137)
    for a, v in ((0, mesh.hy), (1, -mesh.hy), (2, mesh.hx), (3, -mesh.hx)):
        ra = edge_idx[E[:, a]]
        ok = ra >= 0
        tt.add(cell_idx[ok], ra[ok], TERM_CONST, v)
        tt.add(ra[ok], cell_idx[ok], TERM_CONST, v)
    e_row, e_col, tptr, kind, c, k = tt.arrays()
    kl = int(np.max(e_row - e_col)) if len(e_row) else 0
    ku = int(np.max(e_col - e_row)) if len(e_row) else 0

    # Q: star rhs of unit mortar data = -Q c with Q = sigma_out R on the trace
    pos, ndof = _local_mortar_positions(problem, sid)
    qr, qc, qv = [], [], []
    for t in traces:
        R = problem.couplings[(t.iface, sid)].R
        rows = edge_idx[t.edges]
        for m in range(R.shape[0]):
            nz = np.nonzero(R[m])[0]
            qr.append(rows[nz])
            qc.append(np.full(len(nz), pos[(t.iface, 0)][m]))
            qv.append(t.sigma_out * R[m, nz])
    q_ptr, q_row, q_val = _csr(np.concatenate(qc), np.concatenate(qr),
                               np.concatenate(qv), ndof)

    # bar rhs (darcy.py:156-193), realization independent
    bar = np.zeros(n)
    if problem.f_d is not None:
        fx, fy = problem.f_d(mesh.centroids[:, 0], mesh.centroids[:, 1])
        fx = np.broadcast_to(fx, (mesh.n_cells,))
        fy = np.broadcast_to(fy, (mesh.n_cells,))
        half = 0.5 * mesh.hx * mesh.hy
        for col, comp in ((0, fx), (1, fx), (2, fy), (3, fy)):
            r = edge_idx[E[:, col]]
            ok = r >= 0
            np.add.at(bar, r[ok], comp[ok] * half)
    for e, (side, gfun) in pressure.items():
        mid = edge_midpoint(mesh, e)
        gv = 0.0 if gfun is None else float(gfun(mid[0], mid[1]))
        bar[edge_idx[e]] -= OUTWARD_SIGN[side] * gv * mesh.edge_length(e)
    if problem.q_d is not None:
        qv_ = np.broadcast_to(problem.q_d(mesh.centroids[:, 0], mesh.centroids[:, 1]),
                              (mesh.n_cells,))
        bar[cell_idx] -= qv_ * mesh.hx * mesh.hy

    # postprocess: u (edges), p (cells), cv (cells x 2), cp (cells)
    ne, nc = mesh.n_edges, mesh.n_cells
    pr, pc, pv = [], [], []
    kept = np.nonzero(edge_idx >= 0)[0]
    pr.append(kept); pc.append(edge_idx[kept]); pv.append(np.ones(len(kept)))
    pr.append(ne + cells); pc.append(cell_idx); pv.append(np.ones(nc))
    for comp, (a, b) in enumerate(((0, 1), (2, 3))):
        for col in (a, b):
            r = edge_idx[E[:, col]]
            ok = r >= 0
            pr.append(ne + nc + 2 * cells[ok] + comp); pc.append(r[ok])
            pv.append(np.full(int(ok.sum()), 0.5))
    pr.append(ne + 3 * nc + cells); pc.append(cell_idx); pv.append(np.ones(nc))
    nfield = ne + 4 * nc
    p_ptr, p_col, p_val = _csr(np.concatenate(pr), np.concatenate(pc),
                               np.concatenate(pv), nfield)
    layout = [("u", 0, (ne,)), ("p", ne, (nc,)), ("cv", ne + nc, (nc, 2)),
              ("cp", ne + 3 * nc, (nc,))]
    z = np.zeros(0, dtype=np.int64)
    return Pattern(sid, "darcy", n, kl, ku, 0, ndof, nfield, e_row, e_col, tptr, kind,
                   c, k, np.zeros((n, 0)), np.zeros((0, 0)), q_ptr, q_row, q_val, bar,
                   z, np.zeros(1, dtype=np.int64), z.astype(np.int32), np.zeros(0), z,
                   np.zeros(ndof), p_ptr, p_col, p_val, np.zeros(nfield), layout, 0)


# ============================================================= Stokes =====
def _p2_shapes(xi, eta):
    l1 = 1 - xi - eta
    N = np.array([l1 * (2 * l1 - 1), xi * (2 * xi - 1), eta * (2 * eta - 1),
                  4 * l1 * xi, 4 * xi * eta, 4 * eta * l1])
    dN = np.array([[1 - 4 * l1, 1 - 4 * l1], [4 * xi - 1, 0], [0, 4 * eta - 1],
                   [4 * (l1 - xi), -4 * xi], [4 * eta, 4 * xi],
                   [-4 * eta, 4 * (l1 - eta)]], dtype=float)
    return N, dN


def _p1_shapes(xi, eta):
    return np.array([1 - xi - eta, xi, eta])


def taylor_hood_tables(mesh, nu):
    """Element matrices (A11, A22, A12, B1, B2) of both triangle shapes."""
    out = []
    for verts in mesh.tri_vertices[:2]:
        J = np.column_stack([verts[1] - verts[0], verts[2] - verts[0]])
        det = abs(np.linalg.det(J))
        JinvT = np.linalg.inv(J).T
        Kxx, Kyy, Kxy = (np.zeros((6, 6)) for _ in range(3))
        G1, G2 = np.zeros((3, 6)), np.zeros((3, 6))
        for (xi, eta), w in zip(_DUN_P, _DUN_W):
            _, dN = _p2_shapes(xi, eta)
            grad = dN @ JinvT.T
            M = _p1_shapes(xi, eta)
            Kxx += w * det * np.outer(grad[:, 0], grad[:, 0])
            Kyy += w * det * np.outer(grad[:, 1], grad[:, 1])
            Kxy += w * det * np.outer(grad[:, 0], grad[:, 1])
            G1 += w * det * np.outer(M, grad[:, 0])
            G2 += w * det * np.outer(M, grad[:, 1])
        out.append((nu * (2 * Kxx + Kyy), nu * (Kxx + 2 * Kyy), nu * Kxy.T, -G1, -G2))
    return out


def _stokes_boundary(mesh, bcs, traces):
    """Dirichlet dofs/values and traction edges (stokes.py:134-157)."""
    iface_keys = set(tuple(e) for t in traces for e in t.edges)
    dirichlet, stress = {}, []
    for side in SIDES:
        bc = bcs.get(side, StokesBC("velocity"))
        for e in mesh.boundary_edges(side):
            if tuple(e) in iface_keys:
                continue
            if bc.kind == "velocity":
                for node in e:
                    x, y = mesh.p2_xy[node]
                    v = (0.0, 0.0) if bc.value is None else bc.value(x, y)
                    dirichlet[2 * node] = float(v[0])
                    dirichlet[2 * node + 1] = float(v[1])
            elif bc.kind == "stress":
                stress.append((e, bc.value))
            else:
                raise ValueError(f"unknown stokes bc {bc.kind!r}")
    return dirichlet, stress


def _rigid_kernel(mesh, free, A_red_dense_apply, n_udof):
    """Rigid-body modes left in the kernel of the reduced form (stokes.py:276-298)."""
    xy = mesh.p2_xy
    xc, yc = xy.mean(axis=0)
    Z = np.zeros((n_udof, 3))
    Z[0::2, 0] = 1.0
    Z[1::2, 1] = 1.0
    Z[0::2, 2] = -(xy[:, 1] - yc)
    Z[1::2, 2] = xy[:, 0] - xc
    Zf = Z[free]
    nrm = np.linalg.norm(Zf, axis=0)
    nrm[nrm == 0] = 1.0
    Zf = Zf / nrm
    AZ, diag_max = A_red_dense_apply(Zf)
    lam, vecs = np.linalg.eigh(Zf.T @ AZ)
    keep = lam <= 1e-10 * max(diag_max, 1e-30)
    if not keep.any():
        return np.zeros((0, len(free)))
    C = (Zf @ vecs[:, keep]).T
    return C / np.linalg.norm(C, axis=1)[:, None]


def stokes_pattern(problem, sid, k0_offsets, K0_host):
    """Stokes system pattern; BJS terms index the mean-field K buffer.

    k0_offsets[d_sid]: offset of Darcy subdomain d_sid's cells inside the
    concatenated mean-field K buffer the device builds (S3 freezes Stokes at
    y = 0, interface.py:377, 387-388). K0_host (same layout) is used only to
    detect the rigid-body kernel structure (an eigenvalue threshold test,
    stokes.py:276-298); the device evaluates every matrix value itself.
    """
    mesh = problem.meshes[sid]
    bcs = problem.bcs.get(sid, {})
    traces = problem.traces[sid]
    nu, alpha = problem.physics.nu_s, problem.physics.alpha
    n2 = mesh.n_p2
    nud, npr = 2 * n2, mesh.n_p1
    dirichlet, stress = _stokes_boundary(mesh, bcs, traces)
    if not stress and not traces:
        from .errors import SingularOperatorError
        raise SingularOperatorError("stokes subdomain has only velocity data; "
                                    "pressure is undetermined")
    is_dir = np.zeros(nud, dtype=bool)
    g_dir = np.zeros(nud)
    for d, v in dirichlet.items():
        is_dir[d] = True
        g_dir[d] = v
    free = np.nonzero(~is_dir)[0]

    # full velocity-velocity terms (viscous const + BJS 1/sqrt(K)), pressure terms
    tabs = taylor_hood_tables(mesh, nu)
    vv = _TermTable()
    for shape in (0, 1):
        A11, A22, A12, _, _ = tabs[shape]
        nd = mesh.conn_p2[shape::2]
        d1, d2 = 2 * nd, 2 * nd + 1
        # one add per shape, the terms in the order of the loops over
        # (i, j, [11, 22, 12, 21], element): rows[i, j, q, e]
        ne = nd.shape[0]
        R = np.stack([d1.T, d2.T, d1.T, d2.T], axis=1)              # [i, q, e]
        C = np.stack([d1.T, d2.T, d2.T, d1.T], axis=1)              # [j, q, e]
        V = np.stack([A11, A22, A12, A12.T], axis=2)                # [i, j, q]
        rows = np.broadcast_to(R[:, None, :, :], (6, 6, 4, ne))
        cols = np.broadcast_to(C[None, :, :, :], (6, 6, 4, ne))
        vals = np.broadcast_to(V[:, :, :, None], (6, 6, 4, ne))
        vv.add(rows.reshape(-1), cols.reshape(-1), TERM_CONST, vals.reshape(-1))
    bjs_dofs = set()
    if alpha != 0.0:
        for t in traces:
            if t.kind != "sd":
                continue
            d_sid, cells = problem.kl_cells[sid][t.iface]
            tau = np.asarray(t.tangent)
            # one add per trace, the terms in the order of the loops over
            # (edge, a, b, i, j) with the zero tangent products left out
            tri = np.asarray(t.edges, dtype=np.int64)                   # [e, 3]
            if len(tri):
                sb = np.asarray(t.s_breaks, dtype=float)
                Le = sb[1:len(tri) + 1] - sb[:len(tri)]
                kk = k0_offsets[d_sid] + np.asarray(cells, dtype=np.int64)[:len(tri)]
                ab = [(a, b) for a in range(2) for b in range(2) if tau[a] * tau[b] != 0.0]
                if ab:
                    aa = np.array([a for a, _ in ab])
                    bb = np.array([b for _, b in ab])
                    tt = np.array([tau[a] * tau[b] for a, b in ab])
                    shp = (len(tri), len(ab), 3, 3)
                    rows = np.broadcast_to((2 * tri)[:, None, :, None] + aa[None, :, None, None], shp)
                    cols = np.broadcast_to((2 * tri)[:, None, None, :] + bb[None, :, None, None], shp)
                    # nu * alpha * L * mass * ttab, multiplied in the scalar loop's order
                    cf = ((nu * alpha * Le)[:, None, None, None]
                          * np.asarray(P2_EDGE_MASS)[None, None, :, :]) * tt[None, :, None, None]
                    ks = np.broadcast_to(kk[:, None, None, None], shp)
                    vv.add(rows.reshape(-1), cols.reshape(-1), TERM_INV_SQRT_K, cf.reshape(-1),
                           ks.reshape(-1))
                    for a in set(aa.tolist()):
                        bjs_dofs.update((2 * tri + a).reshape(-1).tolist())
    pu = _TermTable()   # B: (p row, u col) constants
    for shape in (0, 1):
        _, _, _, B1, B2 = tabs[shape]
        nd = mesh.conn_p2[shape::2]
        pd = mesh.conn_p1[shape::2]
        # one add per shape, in the order of the loops over (i, j, [1, 2], element)
        ne = nd.shape[0]
        rows = np.broadcast_to(pd.T[:, None, None, :], (3, 6, 2, ne))
        cols = np.broadcast_to(np.stack([2 * nd.T, 2 * nd.T + 1], axis=1)[None, :, :, :],
                               (3, 6, 2, ne))
        vals = np.broadcast_to(np.stack([B1, B2], axis=2)[:, :, :, None], (3, 6, 2, ne))
        pu.add(rows.reshape(-1), cols.reshape(-1), TERM_CONST, vals.reshape(-1))
    vr, vc, vptr, vkind, vcc, vk = vv.arrays()
    prw, pcl, pptr, _, pcc, _ = pu.arrays()
    pval = np.add.reduceat(pcc, pptr[:-1]) if len(pptr) > 1 else np.zeros(0)

    def vv_values(K0):
        vals = np.where(vkind == TERM_INV_SQRT_K, vcc / np.sqrt(K0[vk] if len(K0) else 1.0),
                        vcc)
        return np.add.reduceat(vals, vptr[:-1])

    # kernel detection at the mean-field K (host, structural test only)
    import scipy.sparse as sp
    Aval = vv_values(K0_host)
    A_full = sp.csr_matrix((Aval, (vr, vc)), shape=(nud, nud))
    A_red = A_full[free][:, free]

    def apply_red(Zf):
        return A_red @ Zf, A_red.diagonal().max()

    C = _rigid_kernel(mesh, free, apply_red, nud)
    kdim = C.shape[0]

    # pinned dofs J: complete pivoting on C over dofs without BJS terms
    J = []
    if kdim:
        cand = np.array([j for j, d in enumerate(free) if d not in bjs_dofs])
        Cw = C[:, cand].copy()
        for step in range(kdim):
            sub = np.abs(Cw[step:, :])
            r, cidx = np.unravel_index(np.argmax(sub), sub.shape)
            r += step
            Cw[[step, r]] = Cw[[r, step]]
            J.append(int(cand[cidx]))
            piv = Cw[step, cidx]
            for rr in range(step + 1, kdim):
                Cw[rr] -= Cw[rr, cidx] / piv * Cw[step]
    J_dofs = [int(free[j]) for j in J]

    # band numbering: lattice rows, (ux, uy, p) per node
    vel_idx = -np.ones(nud, dtype=np.int64)
    p_idx = np.empty(npr, dtype=np.int64)
    is_pinned = np.zeros(nud, dtype=bool)
    is_pinned[J_dofs] = True
    nxt = 0
    for ly in range(mesh.my):
        for lx in range(mesh.mx):
            node = ly * mesh.mx + lx
            for a in (0, 1):
                d = 2 * node + a
                if not is_dir[d] and not is_pinned[d]:
                    vel_idx[d] = nxt
                    nxt += 1
            if lx % 2 == 0 and ly % 2 == 0:
                p_idx[(ly // 2) * (mesh.nx + 1) + lx // 2] = nxt
                nxt += 1
    n = nxt
    nb = kdim
    for a, d in enumerate(J_dofs):
        vel_idx[d] = n + a                      # border numbering
    sysidx_u = vel_idx

    # interior entries
    tt = _TermTable()
    keepv = (vel_idx[vr] >= 0) & (vel_idx[vr] < n) & (vel_idx[vc] >= 0) & (vel_idx[vc] < n)
    # expand grouped vv back to per-term lists
    term_entry = np.repeat(np.arange(len(vr)), np.diff(vptr))
    tsel = keepv[term_entry]
    tt.add(vel_idx[vr[term_entry[tsel]]], vel_idx[vc[term_entry[tsel]]], 0, 0.0)
    tt.kind[-1] = vkind[tsel].astype(np.int32)
    tt.c[-1] = vcc[tsel].copy()
    tt.k[-1] = vk[tsel].copy()
    uin = (vel_idx[pcl] >= 0) & (vel_idx[pcl] < n)
    tt.add(p_idx[prw[uin]], vel_idx[pcl[uin]], TERM_CONST, pval[uin])
    tt.add(vel_idx[pcl[uin]], p_idx[prw[uin]], TERM_CONST, pval[uin])
    e_row, e_col, tptr, kind, c, k = tt.arrays()
    kl = int(np.max(e_row - e_col))
    ku = int(np.max(e_col - e_row))

    # rigid-body constraints C (rows over the free velocity dofs): interior part
    # E = C_I^T (n x k), pinned part C_J (k x k) and (C C^T)^-1 (k x k) stacked
    # in G; the device solves the pinned system for a compatible rhs and
    # projects (see band_solve_kernel, section 4)
    E = np.zeros((n, nb))
    G = np.zeros((2 * nb, nb))
    if kdim:
        for r in range(kdim):
            crow = np.zeros(nud)
            crow[free] = C[r]
            inter = (vel_idx >= 0) & (vel_idx < n)
            E[vel_idx[inter], r] = crow[inter]
            for a, d in enumerate(J_dofs):
                G[r, a] = crow[d]
        G[kdim:, :] = np.linalg.inv(C @ C.T)

    # Q and the readout of lifted data on the traces
    pos, ndof = _local_mortar_positions(problem, sid)
    qr, qc, qv = [], [], []
    h_lift = np.zeros(ndof)
    for t in traces:
        R = problem.couplings[(t.iface, sid)].R
        nblk = problem.space.block(t.iface)
        dirs = [np.asarray(t.normal)] + ([np.asarray(t.tangent)] if nblk.n_comp == 2 else [])
        for comp, dvec in enumerate(dirs):
            for a in (0, 1):
                if dvec[a] == 0.0:
                    continue
                dofs = 2 * t.nodes + a
                for m in range(R.shape[0]):
                    nz = np.nonzero(R[m])[0]
                    coef = t.sigma * dvec[a] * R[m, nz]
                    dd = dofs[nz]
                    fr = ~is_dir[dd]
                    qr.append(sysidx_u[dd[fr]])
                    qc.append(np.full(int(fr.sum()), pos[(t.iface, comp)][m]))
                    qv.append(coef[fr])
                    h_lift[pos[(t.iface, comp)][m]] += np.sum(coef[~fr] * g_dir[dd[~fr]])
    # merge duplicate (row, col) pairs (a trace node shared by two edges)
    qr, qc, qv = np.concatenate(qr), np.concatenate(qc), np.concatenate(qv)
    key = qc * (n + nb + 1) + qr
    uk, inv = np.unique(key, return_inverse=True)
    qsum = np.zeros(len(uk))
    np.add.at(qsum, inv, qv)
    q_ptr, q_row, q_val = _csr(uk // (n + nb + 1), uk % (n + nb + 1), qsum, ndof)

    # bar rhs: body force + tractions - A g_dir - B g_dir (stokes.py:305-361)
    Fu = np.zeros(nud)
    if problem.f_s is not None:
        for t_ in range(mesh.n_tri):
            verts = mesh.tri_vertices[t_]
            Jm = np.column_stack([verts[1] - verts[0], verts[2] - verts[0]])
            det = abs(np.linalg.det(Jm))
            nd = mesh.conn_p2[t_]
            for (xi, eta), w in zip(_DUN_P, _DUN_W):
                N, _ = _p2_shapes(xi, eta)
                x, y = verts[0] + Jm @ np.array([xi, eta])
                fx, fy = problem.f_s(x, y)
                Fu[2 * nd] += w * det * fx * N
                Fu[2 * nd + 1] += w * det * fy * N
    for tri, gfun in stress:
        if gfun is None:
            continue
        p0, p1 = mesh.p2_xy[tri[0]], mesh.p2_xy[tri[2]]
        L = np.linalg.norm(p1 - p0)
        for gx, gw in zip(_GL3_X, _GL3_W):
            s_ = 0.5 * (gx + 1)
            x, y = p0 + s_ * (p1 - p0)
            tx, ty = gfun(x, y)
            N = np.array([(1 - s_) * (1 - 2 * s_), 4 * s_ * (1 - s_), s_ * (2 * s_ - 1)])
            for i, node in enumerate(tri):
                Fu[2 * node] += gw * 0.5 * L * tx * N[i]
                Fu[2 * node + 1] += gw * 0.5 * L * ty * N[i]
    # constant part of the lift (viscous), parametrised part (BJS)
    const_terms = vkind == TERM_CONST
    term_row, term_col = vr[term_entry], vc[term_entry]
    lift_c = np.zeros(nud)
    sel = const_terms & is_dir[term_col]
    np.add.at(lift_c, term_row[sel], vcc[sel] * g_dir[term_col[sel]])
    Fu = Fu - lift_c
    Fp = np.zeros(npr)
    selp = is_dir[pcl]
    np.add.at(Fp, prw[selp], pval[selp] * g_dir[pcl[selp]])
    Fp = -Fp
    bar = np.zeros(n + nb)
    fr_nodes = np.nonzero(vel_idx >= 0)[0]
    bar[vel_idx[fr_nodes]] = Fu[fr_nodes]
    bar[p_idx] = Fp
    bt = _TermTable()
    selb = (~const_terms) & is_dir[term_col] & (vel_idx[term_row] >= 0)
    if np.any(selb):
        bt.add(vel_idx[term_row[selb]], 0, 0, 0.0)
        bt.kind[-1] = vkind[selb].astype(np.int32)
        bt.c[-1] = -vcc[selb] * g_dir[term_col[selb]]
        bt.k[-1] = vk[selb].copy()
        if np.any(vel_idx[term_row[selb]] >= n):
            raise ValueError("pinned dofs must not carry BJS lift terms")
    b_row, _, b_tptr, bt_kind, bt_c, bt_k = bt.arrays()

    # postprocess: u (2 n_p2), p (n_p1), cv (n_tri x 2), cp (n_tri)
    ntri = mesh.n_tri
    Nc, _ = _p2_shapes(1 / 3, 1 / 3)
    Mc = _p1_shapes(1 / 3, 1 / 3)
    pr_, pc_, pv_ = [], [], []
    f_lift = np.zeros(nud + npr + 3 * ntri)
    fu = np.nonzero(vel_idx >= 0)[0]
    pr_.append(fu); pc_.append(vel_idx[fu]); pv_.append(np.ones(len(fu)))
    f_lift[:nud] = g_dir
    pr_.append(nud + np.arange(npr)); pc_.append(p_idx); pv_.append(np.ones(npr))
    tri_ids = np.arange(ntri)
    for a in (0, 1):
        for i in range(6):
            dd = 2 * mesh.conn_p2[:, i] + a
            rows = nud + npr + 2 * tri_ids + a
            fr = vel_idx[dd] >= 0
            pr_.append(rows[fr]); pc_.append(vel_idx[dd[fr]]); pv_.append(np.full(int(fr.sum()), Nc[i]))
            np.add.at(f_lift, rows[~fr], Nc[i] * g_dir[dd[~fr]])
    for i in range(3):
        pr_.append(nud + npr + 2 * ntri + tri_ids)
        pc_.append(p_idx[mesh.conn_p1[:, i]])
        pv_.append(np.full(ntri, Mc[i]))
    nfield = nud + npr + 3 * ntri
    p_ptr, p_col, p_val = _csr(np.concatenate(pr_), np.concatenate(pc_),
                               np.concatenate(pv_), nfield)
    layout = [("u", 0, (nud,)), ("p", nud, (npr,)), ("cv", nud + npr, (ntri, 2)),
              ("cp", nud + npr + 2 * ntri, (ntri,))]
    return Pattern(sid, "stokes", n, kl, ku, nb, ndof, nfield, e_row, e_col, tptr, kind, c,
                   k, E, G, q_ptr, q_row, q_val, bar, b_row, b_tptr, bt_kind, bt_c, bt_k,
                   h_lift, p_ptr, p_col, p_val, f_lift, layout, kdim)
