"""Hybridised (SPD) form of the Darcy subdomain problem for the device kernel.

The reference factors the mixed RT0/P0 saddle matrix [A B^T; B 0] per
realization with SuperLU (darcy.py:67-147) and computes the flux basis by
one backsolve per mortar dof (interface.py:218-235). Hybridisation is an
exact algebraic reformulation of the same discrete problem (Arnold-Brezzi):
break normal continuity, introduce one Lagrange multiplier mu_e per edge
(the pressure trace), eliminate (u_T, p_T) cell by cell, and keep an SPD
system H mu = r on the edges. With RT0 on rectangles and the reference's
exact mass matrix (1/3, 1/6 entries, darcy.py:123-131) every cell
contributes K_T * Hhat, where

    Hhat[a][b] = B_a (Mt[a][b] - 3 B_a B_b / (hx^2 + hy^2)) B_b / (nu hx hy),
    Mt = diag([[4,-2],[-2,4]], [[4,-2],[-2,4]]),  B = (hy, -hy, hx, -hx)

over the cell's (west, east, south, north) edges. Interface edges carry the
mortar data as Dirichlet multipliers (mu = lambda_h, the same natural BC
the reference applies, darcy.py:195-207), pressure edges carry g
(darcy.py:178-193), every other edge (interior and no-flow) is unknown.
The flux basis is then a Schur complement: eliminating the unknown edges
from the SPD matrix

    [ H_II        H_IG G        v_b            ]
    [ G^T H_GI    G^T H_GG G    G^T(r_G - H_GP g) ]

leaves [[B, h], ...]: B = G^T (H_GG - H_GI H_II^-1 H_IG) G is the block
of compute_flux_basis and h the bar jump of compute_rhs, with
G = diag(1/|e|) R^T (mortar.py:196-201). Cell-local recovery gives the
fields of postprocess (problem.py:150-158).
"""

from dataclasses import dataclass, field

import numpy as np

from .adapter import OUTWARD_SIGN, SIDES, DarcyBC, cell_edge_table, edge_midpoint

KIND_I, KIND_GAMMA, KIND_P = 0, 1, 2
SMEM_LIMIT = 232448 - 1024        # opt-in dynamic shared memory per CTA on sm_100a


def cell_constants(hx, hy, nu):
    B = np.array([hy, -hy, hx, -hx])
    Mt = np.zeros((4, 4))
    Mt[:2, :2] = [[4.0, -2.0], [-2.0, 4.0]]
    Mt[2:, 2:] = [[4.0, -2.0], [-2.0, 4.0]]
    s2 = hx * hx + hy * hy
    Phat = Mt - 3.0 * np.outer(B, B) / s2
    Hhat = (B[:, None] * Phat * B[None, :]) / (nu * hx * hy)
    return B, Mt, Phat, Hhat, s2


@dataclass
class HybPattern:
    sid: int
    nx: int
    ny: int
    hx: float
    hy: float
    nu: float
    n: int                  # unknown edges
    w: int                  # half bandwidth of H_II in line order
    ndof: int
    nfield: int
    row_edge: np.ndarray    # [n] edge id of unknown r
    edge_kind: np.ndarray   # [n_edges] KIND_*
    edge_idx: np.ndarray    # [n_edges] index within its kind
    edge_cells: np.ndarray  # [n_edges, 2] adjacent cells (-1 none)
    edge_slot: np.ndarray   # [n_edges, 2] local slot (w e s n) in that cell
    edge_noflow: np.ndarray  # [n_edges] 1 on eliminated (no-flow) edges
    cell_edges: np.ndarray  # [n_cells, 4]
    gam_ptr: np.ndarray     # [n_gamma + 1] mortar couplings of interface edges
    gam_d: np.ndarray
    gam_c: np.ndarray       # G[e][d] = R[m(d), t(e)] / |e|
    p_val: np.ndarray       # [n_p] pressure data g on pressure edges
    src_k: np.ndarray       # [n_cells, 4] source rhs, coefficient of K_T
    src_c: np.ndarray       # [n_cells, 4] source rhs, constant part
    cell_f: np.ndarray      # [n_cells, 4] momentum source per local edge
    cell_q: np.ndarray      # [n_cells] integrated mass source q*area
    Hhat: np.ndarray        # [4, 4]
    has_src: bool = False
    field_layout: list = field(default_factory=list)

    @property
    def C(self):
        return self.ndof + 1

    @property
    def Cp(self):
        return (self.ndof + 1 + 7) & ~7

    def layout_for(self, panel):
        """(ws, smem_condense, smem_backsolve, l_doubles, x_doubles) for a panel width."""
        m = self.w + panel
        Cp = self.Cp
        base = m * Cp + Cp * Cp + m * (panel + 4) + panel * (Cp + 4)   # (Yb rows: Cp + 4)
        ws = self.w + 1
        pad = ws + ((8 - ws % 16) % 16)
        if 8 * (m * pad + base) <= SMEM_LIMIT:
            ws = pad
        smem_c = 8 * (m * ws + base)
        smem_b = 8 * (m * Cp + m * (panel + 4) + panel * Cp)
        n_pan = (self.n + panel - 1) // panel
        l_doubles = n_pan * (m * (panel + 4) + panel * Cp)
        return ws, smem_c, smem_b, l_doubles, self.n * Cp

    def panel_entries(self, panel):
        """The assembly entries of the rows entering the condensation window at
        each panel (mfb_darcy.cu condense_kernel), flattened: (pe_ptr [n_pan +
        1], rec [N, 4] {window offset, cell 0, cell 1, terms}, coef [N, 2]).
        The window offset is the entry's destination in the kernel's W | Pb
        shared-memory rows (row r lives in slot r % (w + panel))."""
        T = assembly_tables(self)
        w, n = self.w, self.n
        m = w + panel
        ws = self.layout_for(panel)[0]
        Cp = self.Cp
        n_pan = (n + panel - 1) // panel
        aptr = np.asarray(T["asm_ptr"], dtype=np.int64)
        tptr = np.asarray(T["asm_tptr"], dtype=np.int64)
        cell = np.asarray(T["asm_cell"], dtype=np.int64)
        cf = np.asarray(T["asm_coef"], dtype=np.float64)
        lo = aptr[min(m, n)]                        # entries of rows >= m, in row order
        e = np.arange(lo, aptr[n])
        row = np.repeat(np.arange(n), np.diff(aptr))[e]
        d = np.asarray(T["asm_dest"], dtype=np.int64)[e]
        slot = row % m
        dest = np.where(d <= w, slot * ws + d, m * ws + slot * Cp + (d - w - 1))
        t0, nt = tptr[e], tptr[e + 1] - tptr[e]
        if np.any((nt < 1) | (nt > 2)):
            raise ValueError("assembly entry with other than 1 or 2 terms")
        two = nt == 2
        c1 = np.where(two, cell[np.minimum(t0 + 1, len(cell) - 1)], -1)
        k1 = np.where(two, cf[np.minimum(t0 + 1, len(cf) - 1)], 0.0)
        rec = np.stack([dest, cell[t0], c1, nt], axis=1)
        coef = np.stack([cf[t0], k1], axis=1)
        r0 = np.minimum(np.arange(n_pan + 1) * panel + m, n)
        ptr = aptr[r0] - lo
        return ptr.astype(np.int32), rec.astype(np.int32), coef.astype(np.float64)

    def choose_panel(self):
        for panel in (8,):
            if self.layout_for(panel)[1] <= SMEM_LIMIT:
                return panel
        raise ValueError(f"Darcy subdomain {self.sid}: band {self.w} too wide for shared memory")

    @property
    def algorithmic_flops(self):
        """Work of the condensation as executed: per pivot the trailing lower
        band (w^2), the border panel (2 w C) and the Schur block (C^2)."""
        C = self.ndof + 1
        return float(self.n) * (self.w * self.w + 2.0 * self.w * C + C * C)


def hybrid_pattern(problem, sid):
    mesh = problem.meshes[sid]
    nx, ny = mesh.nx, mesh.ny
    hx, hy = mesh.hx, mesh.hy
    nu = problem.physics.nu_d
    bcs = problem.bcs.get(sid, {})
    traces = problem.traces[sid]
    ne, nc = mesh.n_edges, mesh.n_cells
    kind = np.full(ne, KIND_I, dtype=np.int32)
    idx = -np.ones(ne, dtype=np.int64)
    noflow = np.zeros(ne, dtype=np.int32)
    # interface edges, in trace order
    gam_edges, gam_rows = [], []
    for t in traces:
        R = problem.couplings[(t.iface, sid)].R
        pos = _mortar_positions(problem, sid)[t.iface]
        for j, e in enumerate(t.edges):
            e = int(e)
            kind[e] = KIND_GAMMA
            idx[e] = len(gam_edges)
            L = mesh.edge_length(e)
            nz = np.nonzero(R[:, j])[0]
            gam_edges.append(e)
            gam_rows.append((pos[nz], R[nz, j] / L))
    p_vals = []
    for side in SIDES:
        bc = bcs.get(side, DarcyBC("noflow"))
        for e in mesh.boundary_edges(side):
            e = int(e)
            if kind[e] == KIND_GAMMA:
                continue
            if bc.kind == "noflow":
                noflow[e] = 1
            elif bc.kind == "pressure":
                kind[e] = KIND_P
                idx[e] = len(p_vals)
                mid = edge_midpoint(mesh, e)
                p_vals.append(0.0 if bc.value is None else float(bc.value(mid[0], mid[1])))
            else:
                raise ValueError(f"unknown darcy bc {bc.kind!r}")
    if not p_vals and not gam_edges:
        from .errors import SingularOperatorError
        raise SingularOperatorError("darcy subdomain has no pressure data and no "
                                    "interface; pressure is undetermined")
    # unknown ordering: per line j, h-edges(j) then v-edges(row j)
    row_edge = []
    for j in range(ny + 1):
        for ix in range(nx):
            e = mesh.hedge(ix, j)
            if kind[e] == KIND_I:
                row_edge.append(e)
        if j < ny:
            for ix in range(nx + 1):
                e = mesh.vedge(ix, j)
                if kind[e] == KIND_I:
                    row_edge.append(e)
    row_edge = np.array(row_edge, dtype=np.int64)
    idx[row_edge] = np.arange(len(row_edge))
    n = len(row_edge)
    CE = cell_edge_table(mesh)
    ecell = -np.ones((ne, 2), dtype=np.int64)
    eslot = -np.ones((ne, 2), dtype=np.int64)
    for c in range(nc):
        for a in range(4):
            e = CE[c, a]
            k = 0 if ecell[e, 0] < 0 else 1
            ecell[e, k] = c
            eslot[e, k] = a
    # half bandwidth over couplings between unknowns
    w = 0
    for c in range(nc):
        ii = idx[CE[c]][kind[CE[c]] == KIND_I]
        if len(ii):
            w = max(w, int(ii.max() - ii.min()))
    B, Mt, Phat, Hhat, s2 = cell_constants(hx, hy, nu)
    # sources (darcy.py:156-193): f per local edge (midpoint rule), q integrated
    cell_f = np.zeros((nc, 4))
    cell_q = np.zeros(nc)
    has_src = False
    if problem.f_d is not None:
        fx, fy = problem.f_d(mesh.centroids[:, 0], mesh.centroids[:, 1])
        half = 0.5 * hx * hy
        cell_f[:, 0] = cell_f[:, 1] = np.broadcast_to(fx, (nc,)) * half
        cell_f[:, 2] = cell_f[:, 3] = np.broadcast_to(fy, (nc,)) * half
        has_src = True
    if problem.q_d is not None:
        cell_q[:] = np.broadcast_to(problem.q_d(mesh.centroids[:, 0], mesh.centroids[:, 1]),
                                    (nc,)) * hx * hy
        has_src = True
    # continuity rhs r_T = C P f + (B o B) q / (2 s2), P = K/(nu A) Phat, C = -diag(B)
    src_k = -(B[None, :] * (cell_f @ Phat.T)) / (nu * hx * hy)
    src_c = (B * B)[None, :] * cell_q[:, None] / (2.0 * s2)
    gam_ptr = np.cumsum([0] + [len(r[0]) for r in gam_rows]).astype(np.int64)
    gam_d = np.concatenate([r[0] for r in gam_rows]) if gam_rows else np.zeros(0, dtype=np.int64)
    gam_c = np.concatenate([r[1] for r in gam_rows]) if gam_rows else np.zeros(0)
    ndof = sum(problem.space.block(g.index).n_dof for g in problem.layout.interfaces_of(sid))
    layout = [("u", 0, (ne,)), ("p", ne, (nc,)), ("cv", ne + nc, (nc, 2)),
              ("cp", ne + 3 * nc, (nc,))]
    return HybPattern(sid, nx, ny, hx, hy, nu, n, w, ndof, ne + 4 * nc, row_edge, kind, idx,
                      ecell, eslot, noflow, CE, gam_ptr, gam_d.astype(np.int64), gam_c,
                      np.array(p_vals), src_k, src_c, cell_f, cell_q, Hhat, has_src, layout)


def _mortar_positions(problem, sid):
    out, start = {}, 0
    for g in problem.layout.interfaces_of(sid):
        b = problem.space.block(g.index)
        out[g.index] = start + np.arange(b.n_scalar) * b.n_comp
        start += b.n_dof
    return out


# ------------------------------------------------------------------ CPU model
def dense_model(hp, K):
    """Dense H_II, V = [H_IG G | v_b], Z (CPU reference of the device kernel)."""
    K = np.asarray(K, dtype=float)
    n, nd = hp.n, hp.ndof
    C = nd + 1
    H = np.zeros((n, n))
    V = np.zeros((n, C))
    Z = np.zeros((C, C))
    nG = len(hp.gam_ptr) - 1

    def gvec(e):
        g = np.zeros(C)
        gi = hp.edge_idx[e]
        sl = slice(hp.gam_ptr[gi], hp.gam_ptr[gi + 1])
        np.add.at(g, hp.gam_d[sl], hp.gam_c[sl])
        return g

    for c in range(len(K)):
        E = hp.cell_edges[c]
        Hc = K[c] * hp.Hhat
        r = K[c] * hp.src_k[c] + hp.src_c[c]
        for a in range(4):
            ea, ka = E[a], hp.edge_kind[E[a]]
            for b in range(4):
                eb, kb = E[b], hp.edge_kind[E[b]]
                h = Hc[a, b]
                if ka == KIND_I and kb == KIND_I:
                    H[hp.edge_idx[ea], hp.edge_idx[eb]] += h
                elif ka == KIND_I and kb == KIND_GAMMA:
                    V[hp.edge_idx[ea]] += h * gvec(eb)
                elif ka == KIND_I and kb == KIND_P:
                    V[hp.edge_idx[ea], nd] -= h * hp.p_val[hp.edge_idx[eb]]
                elif ka == KIND_GAMMA and kb == KIND_GAMMA:
                    Z[:nd, :nd] += h * np.outer(gvec(ea), gvec(eb))[:nd, :nd]
                elif ka == KIND_GAMMA and kb == KIND_P:
                    Z[:nd, nd] -= h * gvec(ea)[:nd] * hp.p_val[hp.edge_idx[eb]]
            if ka == KIND_I:
                V[hp.edge_idx[ea], nd] += r[a]
            elif ka == KIND_GAMMA:
                Z[:nd, nd] += r[a] * gvec(ea)[:nd]
    del nG
    return H, V, Z


def condense(hp, K):
    """(B, h, X) with X = H_II^-1 V."""
    H, V, Z = dense_model(hp, K)
    X = np.linalg.solve(H, V) if hp.n else np.zeros_like(V)
    S = Z - V.T @ X
    nd = hp.ndof
    return S[:nd, :nd], S[:nd, nd], X


def recover_fields(hp, K, X):
    """Fields (u, p, cv, cp) of the bar solution and of each unit mortar column.

    Returns (Fb, M) with fields(lambda) = Fb - M lambda, matching the generic
    pattern's postprocess layout."""
    K = np.asarray(K, dtype=float)
    nd = hp.ndof
    ne, nc = len(hp.edge_kind), len(K)
    B, Mt, Phat, Hhat, s2 = cell_constants(hp.hx, hp.hy, hp.nu)
    out = np.zeros((ne + 4 * nc, nd + 1))   # columns: star(e_d) ..., bar
    for c in range(nc):
        E = hp.cell_edges[c]
        mu = np.zeros((4, nd + 1))
        for a in range(4):
            e = E[a]
            k = hp.edge_kind[e]
            if k == KIND_I:
                mu[a, :nd] = -X[hp.edge_idx[e], :nd]
                mu[a, nd] = X[hp.edge_idx[e], nd]
            elif k == KIND_GAMMA:
                gi = hp.edge_idx[e]
                sl = slice(hp.gam_ptr[gi], hp.gam_ptr[gi + 1])
                np.add.at(mu[a], hp.gam_d[sl], hp.gam_c[sl])
            else:
                mu[a, nd] = hp.p_val[hp.edge_idx[e]]
        kap = K[c] / (hp.nu * hp.hx * hp.hy)
        f = np.zeros((4, nd + 1))
        f[:, nd] = hp.cell_f[c]
        q = np.zeros(nd + 1)
        q[nd] = hp.cell_q[c]
        g = f + B[:, None] * mu                                  # f - C mu
        u = kap * (Phat @ g) - np.outer(B, q) / (2.0 * s2)
        p = ((B @ f) + (B * B) @ mu) / (2.0 * s2) + q / (12.0 * kap * s2)
        for a in range(4):
            e = E[a]
            if hp.edge_cells[e, 0] == c:
                out[e] = 0.0 if hp.edge_noflow[e] else u[a]
        out[ne + c] = p
        out[ne + nc + 2 * c] = 0.5 * (u[0] + u[1])
        out[ne + nc + 2 * c + 1] = 0.5 * (u[2] + u[3])
        out[ne + 3 * nc + c] = p
    return out[:, nd], -out[:, :nd]


def assembly_tables(hp):
    """Term tables the device uses to assemble window rows and the border block.

    Row table (CSR over unknown rows r): entries with a destination
    `dest` = c - r + w for H_II[r][c] (c <= r, inside the band) or
    w + 1 + d for border column d (d = ndof is the bar column); each entry
    is a short list of terms coef * K[cell] (cell >= 0) or coef (cell = -1),
    summed in list order. Z table: entries d1 * (ndof+1) + d2 of the initial
    border block with terms of the same form.
    """
    nd = hp.ndof
    w = hp.w
    rows = {}          # r -> {dest: [(cell, coef)]}
    zent = {}          # (d1, d2) -> [(cell, coef)]

    def gvec(e):
        gi = hp.edge_idx[e]
        sl = slice(hp.gam_ptr[gi], hp.gam_ptr[gi + 1])
        return list(zip(hp.gam_d[sl].tolist(), hp.gam_c[sl].tolist()))

    for c in range(len(hp.cell_q)):
        E = hp.cell_edges[c]
        for a in range(4):
            ea, ka = int(E[a]), hp.edge_kind[E[a]]
            if ka == KIND_I:
                r = int(hp.edge_idx[ea])
                ent = rows.setdefault(r, {})
                for b in range(4):
                    eb, kb = int(E[b]), hp.edge_kind[E[b]]
                    h = float(hp.Hhat[a, b])
                    if kb == KIND_I:
                        col = int(hp.edge_idx[eb])
                        if col <= r:
                            ent.setdefault(col - r + w, []).append((c, h))
                    elif kb == KIND_GAMMA:
                        for d, gc in gvec(eb):
                            ent.setdefault(w + 1 + d, []).append((c, h * gc))
                    else:
                        ent.setdefault(w + 1 + nd, []).append(
                            (c, -h * float(hp.p_val[hp.edge_idx[eb]])))
                if hp.has_src:
                    ent.setdefault(w + 1 + nd, []).append((c, float(hp.src_k[c, a])))
                    ent[w + 1 + nd].append((-1, float(hp.src_c[c, a])))
            elif ka == KIND_GAMMA:
                for d1, g1 in gvec(ea):
                    for b in range(4):
                        eb, kb = int(E[b]), hp.edge_kind[E[b]]
                        h = float(hp.Hhat[a, b])
                        if kb == KIND_GAMMA:
                            for d2, g2 in gvec(eb):
                                zent.setdefault((d1, d2), []).append((c, g1 * h * g2))
                        elif kb == KIND_P:
                            zent.setdefault((d1, nd), []).append(
                                (c, -g1 * h * float(hp.p_val[hp.edge_idx[eb]])))
                    if hp.has_src:
                        zent.setdefault((d1, nd), []).append((c, g1 * float(hp.src_k[c, a])))
                        zent[(d1, nd)].append((-1, g1 * float(hp.src_c[c, a])))

    ptr, dest, tptr, tcell, tcoef = [0], [], [0], [], []
    for r in range(hp.n):
        for dd in sorted(rows.get(r, {})):
            dest.append(dd)
            for cell, coef in rows[r][dd]:
                tcell.append(cell)
                tcoef.append(coef)
            tptr.append(len(tcell))
        ptr.append(len(dest))
    zdest, ztptr, zcell, zcoef = [], [0], [], []
    for (d1, d2) in sorted(zent):
        zdest.append(d1 * (nd + 1) + d2)
        for cell, coef in zent[(d1, d2)]:
            zcell.append(cell)
            zcoef.append(coef)
        ztptr.append(len(zcell))
    return {k: np.asarray(v) for k, v in dict(
        asm_ptr=ptr, asm_dest=dest, asm_tptr=tptr, asm_cell=tcell, asm_coef=tcoef,
        z_dest=zdest, z_tptr=ztptr, z_cell=zcell, z_coef=zcoef).items()}
