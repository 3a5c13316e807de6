"""Work tables of the cluster CG (csrc/mfb_cg_cluster.cu).

The interface CG of a large interface (cfg4: n_lambda = 2,720 over 128
subdomains) runs NP collocation points per thread-block CLUSTER of C CTAs.
The subdomains are split into C geometric parts (sorted by block centre x,
then y, cut into chunks of equal sum N_dof^2): CTA c of a cluster applies
the flux-basis blocks of its part only, and keeps the CG vectors of the
mortar dofs it OWNS on chip -- a dof is owned by the part of its first
(lower-sid) side, interface.cg_tasks' `sides[d].x`.

Per rank c the tables say:

* owned dofs (ascending global id) = local indices 0..n_own-1, then the halo
  dofs (used by a block of the part, owned elsewhere, ascending): the rows
  of p in shared memory;
* tasks: runs of <= 8 dofs of one interface (cg_tasks' runs). A run whose two
  sides are both in the part is computed whole (S p = lower row + upper row,
  basis_apply's order, interface.py:238-247); a run cut by the partition is
  computed as the lower row by the owner and as the upper row by the other
  part, which stores it into the owner's cut buffer (DSMEM); the owner adds
  it (lower + upper: the same single addition);
* the column map of every block of the part (local p row of each column);
* per owned dof the one peer (rank, local row) that holds it as halo, which
  the owner updates with every new p (DSMEM).

`emulate_apply` runs the tables on the host (numpy) and is what the CPU
tests check against the direct S p.
"""

import numpy as np

HDR = 16        # ints per rank header (see cluster_tables)


def partition(n_sub, centers, cost, C):
    """Sids -> part (0..C-1): ordered by centre (x, then y), contiguous chunks
    with equal shares of `cost`; whole columns of blocks (equal centre x) stay
    in one part when there are at least C columns (straight cuts)."""
    centers = np.asarray(centers, dtype=np.float64)
    cost = np.asarray(cost, dtype=np.float64)
    ux, col = np.unique(np.round(centers[:, 0], 12), return_inverse=True)
    if len(ux) >= C:
        ccost = np.bincount(col, weights=cost, minlength=len(ux))
        cum = np.cumsum(ccost) - 0.5 * ccost
        cpart = np.minimum((cum * C / max(ccost.sum(), 1e-300)).astype(np.int64), C - 1)
        if len(np.unique(cpart)) == C:
            return cpart[col]
    order = np.lexsort((centers[:, 1], centers[:, 0]))
    cost = np.asarray(cost, dtype=np.float64)[order]
    cum = np.cumsum(cost) - 0.5 * cost
    part = np.empty(n_sub, dtype=np.int64)
    part[order] = np.minimum((cum * C / max(cost.sum(), 1e-300)).astype(np.int64), C - 1)
    return part


def cluster_tables(n_sub, ndof, dof_ptr, dof_map, n_lambda, region, centers, C, NP,
                   tasks, sides, pk_base, pk_size):
    """Per-rank tables of the cluster CG.

    tasks / sides / pk_size: interface.cg_tasks output (the interface runs of
    <= 8 dofs and their two sides' strip offsets); pk_base: per-sid base of the
    packed pool (loc 0). Returns dict with `hdr` [C, HDR] and `tab` (int32, all
    ranks' tables concatenated) plus sizes for the launch.

    Work is organised by UNITS: one subdomain block of the rank in one of two
    passes. Pass 1 applies the lower-side strips of its runs (S p rows := row
    product), pass 2 the upper-side strips (S p rows += row product, or into
    the owner's cut buffer when the run's owner is another rank): lower +
    upper, basis_apply's single addition. A unit loads the block's B operand
    (p at its columns) once and streams its strips' A fragments.

    hdr[c] = {n_own, n_used, n_units, n_cut, n_cm, off_own, off_peer, off_unit,
    off_cm, off_cut, n_strips, off_strip, n_units_pass1, 0, 0, 0}; in tab:
      own   [n_own]       global dof of owned row d
      peer  [2 n_own]     (rank, local row) of the peer holding it as halo, or (-1, -1)
      unit  [8 n_units]   {nd, region, packed block size, column-map offset,
                           strips, first strip, pass, cost}; pass-1 units first,
                           each pass most expensive first
      cm    [n_cm]        local p row of every column of the part's blocks
      cut   [n_cut]       owned row of cut row q (remote upper rows land there)
      strip [4 n_strips]  {packed offset of the strip (loc 0), R | kind << 8 |
                           owner << 12, destination row, 0}; kind 1: pass-1
                           rows (:=), 2: pass-2 rows (+=), 6: pass-2 rows to the
                           cut buffer of rank `owner` (destination = cut row)
    """
    ndof = np.asarray(ndof, dtype=np.int64)
    dof_ptr = np.asarray(dof_ptr, dtype=np.int64)
    dof_map = np.asarray(dof_map, dtype=np.int64)
    cost = ndof.astype(np.float64) ** 2
    part = partition(n_sub, centers, cost, C)
    first = np.asarray(sides)[:, 0].astype(np.int64)
    owner = part[first]
    own = [np.nonzero(owner == c)[0] for c in range(C)]
    used = []
    for c in range(C):
        u = np.unique(np.concatenate([dof_map[dof_ptr[s]:dof_ptr[s + 1]]
                                      for s in range(n_sub) if part[s] == c] or [np.zeros(0, int)]))
        halo = np.setdiff1d(u, own[c])
        used.append(np.concatenate([own[c], halo]))
    loc = [dict() for _ in range(C)]
    for c in range(C):
        for k, d in enumerate(used[c]):
            loc[c][int(d)] = k
    peer = [np.full((len(own[c]), 2), -1, dtype=np.int64) for c in range(C)]
    for c in range(C):
        for d in used[c][len(own[c]):]:
            oc = int(owner[d])
            peer[oc][loc[oc][int(d)]] = (c, loc[c][int(d)])
    cm, cm_off = [[] for _ in range(C)], {}
    for s in range(n_sub):
        c = int(part[s])
        cm_off[s] = len(cm[c])
        cm[c].extend(loc[c][int(d)] for d in dof_map[dof_ptr[s]:dof_ptr[s + 1]])
    cut = [[] for _ in range(C)]
    strips = {}                        # (sid, pass) -> [strip records]
    for t in np.asarray(tasks).reshape(-1, 4):
        d0, so_lo, so_up, meta = (int(v) for v in t)
        i, j, R = meta & 0xfff, ((meta >> 12) & 0xfff) - 1, meta >> 24
        ci = int(part[i])
        dst = loc[ci][d0]
        strips.setdefault((i, 1), []).append((int(pk_base[i]) + so_lo, R, 1, ci, dst))
        if j < 0:
            continue
        if part[j] == ci:
            strips.setdefault((j, 2), []).append((int(pk_base[j]) + so_up, R, 2, ci, dst))
        else:
            q0 = len(cut[ci])
            cut[ci].extend(range(dst, dst + R))
            strips.setdefault((j, 2), []).append((int(pk_base[j]) + so_up, R, 6, ci, q0))
    hdr = np.zeros((C, HDR), dtype=np.int64)
    chunks, off = [], 0
    for c in range(C):
        units, srec = [], []
        for ps in (1, 2):
            ul = []
            for s in range(n_sub):
                if part[s] != c or (s, ps) not in strips:
                    continue
                sl = sorted(strips[(s, ps)], key=lambda r: r[0])
                ul.append((int(ndof[s]) * len(sl), s, sl))
            ul.sort(key=lambda u: -u[0])
            for cst, s, sl in ul:
                units.append((int(ndof[s]), int(region[s]), int(pk_size[s]), cm_off[s], len(sl),
                              len(srec), ps, cst))
                for pk, R, kind, ow, dst in sl:
                    srec.append((pk, R | (kind << 8) | (ow << 12), dst, 0))
        n1 = sum(1 for u in units if u[6] == 1)
        urec = np.array(units, dtype=np.int64).reshape(-1, 8)
        srec = np.array(srec, dtype=np.int64).reshape(-1, 4)
        parts = [own[c], peer[c].ravel(), urec.ravel(), np.asarray(cm[c], dtype=np.int64),
                 np.asarray(cut[c], dtype=np.int64), srec.ravel()]
        offs = []
        for a in parts:
            pad = (-off) % 4                 # int2 / int4 loads: 16-byte aligned starts
            if pad:
                chunks.append(np.zeros(pad, dtype=np.int64))
                off += pad
            offs.append(off)
            chunks.append(a.astype(np.int64))
            off += len(a)
        hdr[c] = (len(own[c]), len(used[c]), len(urec), len(cut[c]), len(cm[c]),
                  offs[0], offs[1], offs[2], offs[3], offs[4], len(srec), offs[5], n1, 0, 0, 0)
    tab = np.concatenate(chunks) if chunks else np.zeros(0, dtype=np.int64)
    if tab.size and (tab.max() >= 2 ** 31 or tab.min() < -1):
        raise ValueError("cluster CG tables exceed int32")
    n_own_max, n_used_max = int(hdr[:, 0].max()), int(hdr[:, 1].max())
    n_cut_max = int(hdr[:, 3].max())
    return {"hdr": hdr.astype(np.int32), "tab": tab.astype(np.int32), "part": part,
            "n_own_max": n_own_max, "n_used_max": n_used_max, "n_cut_max": n_cut_max,
            "n_cm_max": int(hdr[:, 4].max()), "n_unit_max": int(hdr[:, 2].max()),
            "n_strip_max": int(hdr[:, 10].max()), "C": C, "NP": NP}


def emulate_apply(ct, block, strip_of, P):
    """Host emulation of one S p through the tables: block(sid) -> dense
    [nd, nd] block (the slot's local realization), strip_of(packed offset)
    -> (sid, first row), P [n_lambda, NP].
    Returns S p [n_lambda, NP] assembled the way the kernel does (pass 1 rows
    :=, pass 2 rows += or through the owner's cut buffer)."""
    hdr, tab, C = ct["hdr"].astype(np.int64), ct["tab"].astype(np.int64), ct["C"]
    Sp = np.full_like(P, np.nan)
    cbuf = [np.zeros((max(int(hdr[c, 3]), 1), P.shape[1])) for c in range(C)]
    pl = []
    for c in range(C):
        n_own, n_used = int(hdr[c, 0]), int(hdr[c, 1])
        own = tab[hdr[c, 5]:hdr[c, 5] + n_own]
        peer = tab[hdr[c, 6]:hdr[c, 6] + 2 * n_own].reshape(-1, 2)
        pl.append((own, peer, np.zeros((n_used, P.shape[1]))))
    for c in range(C):                  # owned rows, halo rows through the owners
        own, peer, p = pl[c]
        p[:len(own)] = P[own]
        for k, (r, row) in enumerate(peer):
            if r >= 0:
                pl[r][2][row] = P[own[k]]
    spl = []
    for c in range(C):
        n_own = int(hdr[c, 0])
        p = pl[c][2]
        sp = np.full((n_own, P.shape[1]), np.nan)
        cm = tab[hdr[c, 8]:hdr[c, 8] + hdr[c, 4]]
        units = tab[hdr[c, 7]:hdr[c, 7] + 8 * hdr[c, 2]].reshape(-1, 8)
        srec = tab[hdr[c, 11]:hdr[c, 11] + 4 * hdr[c, 10]].reshape(-1, 4)
        assert np.all(units[:hdr[c, 12], 6] == 1) and np.all(units[hdr[c, 12]:, 6] == 2)
        for nd, reg, psz, cmo, ns, so, ps, _ in units:       # pass 1 units, then pass 2
            B = None
            for pk, w, dst, _ in srec[so:so + ns]:
                R, kind, ow = w & 0xff, (w >> 8) & 0xf, w >> 12
                sid, r0 = strip_of(pk)
                B = block(sid)
                assert B.shape[0] == nd
                rows = B[r0:r0 + R] @ p[cm[cmo:cmo + nd]]
                if kind == 1:
                    sp[dst:dst + R] = rows
                elif kind == 2:
                    sp[dst:dst + R] = sp[dst:dst + R] + rows
                else:
                    cbuf[ow][dst:dst + R] = rows
        spl.append(sp)
    for c in range(C):
        n_cut = int(hdr[c, 3])
        cut = tab[hdr[c, 9]:hdr[c, 9] + n_cut]
        for q, d in enumerate(cut):
            spl[c][d] = spl[c][d] + cbuf[c][q]
        Sp[pl[c][0]] = spl[c]
    assert not np.isnan(Sp).any(), "a dof was not produced by any rank"
    return Sp
