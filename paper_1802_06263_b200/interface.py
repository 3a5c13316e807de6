"""Drop-in `run_method` for Methods S3, S2 and S1 on one B200.

Same signature, return type and error behaviour as the reference's
`sdmortar.interface.run_method` (interface.py:288-346): a `RunResult` with
`moments` {key: (mean, var)} over the keys "lambda" and "{sid}:{u,p,cv,cp}",
per-subdomain `SolveStats`, the per-point mortar solutions `lambdas` and CG
residual histories `residuals`. Underneath, every piece of compute runs on
the device through the C ABI (include/mfb.h):

  1. KL kernel: K for every local realization of every region (+ mean field)
  2. one batched launch assembles, factors and solves every (subdomain,
     local realization) system against all mortar columns and the bar rhs,
     then extracts the flux-basis blocks, bar jumps and field responses
  3. one batched CG launch solves all collocation points concurrently
  4. moment kernels (lambda streamed in realization order; fields through
     per-group shifted statistics)

Method S2 (the deterministic MFB) runs the same kernels
with one system per (subdomain, global realization). Method S1 (matrix-free,
8f row 2) factors the same per-realization systems, keeps the factors, and
applies the interface operator by a batched star solve per CG iteration
(mfb_systems_apply + mfb_s1_cg_step); its moments stream every point's
fields in realization order. There is no CPU fallback.
"""

import ctypes
from collections.abc import Sequence
import logging
import time
from dataclasses import dataclass, field

import sys

import numpy as np

from . import _lib
from .adapter import mode_table
from .errors import ConvergenceError, NativeLibraryError, SingularOperatorError, SizeCapError
from .plan import DevicePlan, _dev, _ptr

log = logging.getLogger(__name__)

METHODS = ("S1", "S2", "S3")
_PLAN_CACHE = {}
PLAN_CACHE_SIZE = 8         # device plans kept (least recently used evicted)
# Sweep states of different plans may share their large device buffers (the
# basis pool, field responses, factor work, K): sweeps that go through
# run_method rebuild them in every call, so plans of the same problem on
# different grids (e.g. batches of one collocation grid) then cost one set of
# buffers instead of one each. Off by default: a caller holding two engines'
# results at once must keep them separate. A sweep that would read a buffer
# another state has since overwritten raises NativeLibraryError instead.
SHARE_SCRATCH = False
_SHARED = {}
_OWNER = {}


def _scratch(name, numel, dtype):
    """Device buffer for a sweep state: its own, or with SHARE_SCRATCH a view
    of one buffer per (name, dtype) shared by every state."""
    import torch
    numel = int(numel)
    if not SHARE_SCRATCH:
        return torch.empty(numel, dtype=dtype, device="cuda")
    t = _SHARED.get((name, dtype))
    if t is None or t.numel() < numel:
        _SHARED.pop((name, dtype), None)
        t = torch.empty(numel, dtype=dtype, device="cuda")
        _SHARED[(name, dtype)] = t
    return t[:numel]


def _claim(st, *names):
    """st's results now live in the shared buffers `names`."""
    if SHARE_SCRATCH:
        for n in names:
            _OWNER[n] = st


def _check_owner(st, *names):
    if SHARE_SCRATCH:
        for n in names:
            if _OWNER.get(n, st) is not st:
                raise NativeLibraryError(
                    f"shared sweep buffer '{n}' holds another sweep's results "
                    f"(SHARE_SCRATCH): rebuild this engine's bases first")
WORK_BUDGET_BYTES = 16 << 30
N_SMS = 148                 # B200
BAND_GROUP_MAX = 16         # CTAs per banded system (cooperative launch)
S1_FIELD_BYTES_MAX = 32 << 30   # S1 keeps every realization's fields for the moments
S1_CHUNK_REALIZATIONS = None    # S1 realizations per chunk (None: as many as fit)
CLUSTER_SHAPES = ((4, 16), (8, 16), (2, 8), (4, 8))   # (CTAs per cluster, points) to try
SYMMETRIZE_BAND_BLOCKS = True   # basis blocks from the banded LU: B <- (B + B^T) / 2
MULTI_STREAM = True         # multi-point CG: S p streamed over per-warp pass lists
MULTI_CHUNKS = True         # multi-point CG: reflection-family point order + chunked claims
MULTI_TAIL = None           # points claimed singly at the sweep's end (None: one per slot, 8 x CTAs)
HIST_SEG = 1024             # residual-history segment (large-interface CG kernels)
_HIST_POOL = {}             # the last solve's segment pool, reused when unreferenced
PINNED_HIST_BYTES_MAX = 8 << 30   # residual histories up to this size come back in pinned memory
_HIST_STAGE_DOUBLES = 32 << 20    # staging chunk (256 MB) of the pageable path
MOMENTS_MAX_NDOF = 64       # mfb_group_stats / mfb_group_fields block limit (mfb.h)
KL_MAX_TERM = 64            # mfb_kl_realize_batched terms per region (mfb.h)


@dataclass
class SolveStats:
    """Per-subdomain counters in the reference's semantics (interface.py:35-77).

    Backsolve counts are the reference's S3 identities (interface.py:14-16):
    N_dof_i N_loc(i) basis solves + 2 N_real (bar + recovery), one
    factorization per local realization; the device realises the same
    solves as batched multi-RHS eliminations.
    """

    method: str
    n_sub: int
    factorizations: np.ndarray
    backsolves: np.ndarray
    basis_backsolves: np.ndarray
    cg_iters: list = field(default_factory=list)
    wall_seconds: np.ndarray = None
    n_real: int = 0

    @classmethod
    def new(cls, method, n_sub):
        z = lambda: np.zeros(n_sub, dtype=int)
        return cls(method, n_sub, z(), z(), z(), wall_seconds=np.zeros(n_sub))

    @property
    def cg_iters_total(self):
        return int(sum(self.cg_iters))

    def rows(self):
        return [{"method": self.method, "subdomain": sid,
                 "factorizations": int(self.factorizations[sid]),
                 "backsolves": int(self.backsolves[sid]),
                 "basis_backsolves": int(self.basis_backsolves[sid]),
                 "cg_iters_total": self.cg_iters_total, "n_real": self.n_real,
                 "wall_seconds": float(self.wall_seconds[sid])}
                for sid in range(self.n_sub)]


@dataclass
class RunResult:
    moments: dict
    stats: SolveStats
    lambdas: list
    residuals: list
    grid: object
    timings: dict = field(default_factory=dict)


class ResidualHistories(Sequence):
    """Per-point CG residual histories (reference: `RunResult.residuals`, a
    list of per-point lists, interface.py:284,335) kept as one flat array.

    Indexing returns the point's history as a Python list, like the
    reference; the flat storage keeps a cfg4-scale sweep (54,273 points x
    ~13k iterations) at 8 bytes per entry instead of a Python float each.
    """

    def __init__(self, flat, iters, padded=None):
        self.flat = flat
        self.iters = np.asarray(iters, dtype=np.int64)
        self.offsets = np.concatenate([[0], np.cumsum(self.iters)])
        self._padded = padded

    @classmethod
    def from_padded(cls, padded, iters):
        """Histories left in the [points, cap] array the device wrote (row k
        valid up to iters[k]): no repacking; `flat` is built on first use."""
        h = cls.__new__(cls)
        h.iters = np.asarray(iters, dtype=np.int64)
        h._padded = padded
        h._flat = None
        return h

    @classmethod
    def from_segments(cls, pool, seg_tab, iters, seg):
        """Histories in the segment pool the cluster CG wrote: point k's
        entry i at pool[seg_tab[k, i // seg] * seg + i % seg]."""
        h = cls.__new__(cls)
        h.iters = np.asarray(iters, dtype=np.int64)
        h._padded = None
        h._seg = (pool, seg_tab, int(seg))
        return h

    def __getattr__(self, name):          # lazy flat/offsets of a padded or segmented store
        if name in ("flat", "offsets") and self.__dict__.get("_seg") is not None:
            it = self.iters
            self.offsets = np.concatenate([[0], np.cumsum(it)])
            self.flat = (np.concatenate([self.array(k) for k in range(len(it))])
                         if len(it) else np.zeros(0))
            return self.__dict__[name]
        if name in ("flat", "offsets") and self.__dict__.get("_padded") is not None:
            it = self.iters
            mask = np.arange(self._padded.shape[1])[None, :] < it[:, None]
            self.flat = self._padded[mask]
            self.offsets = np.concatenate([[0], np.cumsum(it)])
            return self.__dict__[name]
        raise AttributeError(name)

    def __len__(self):
        return len(self.iters)

    def __getitem__(self, k):
        if isinstance(k, slice):
            return [self[j] for j in range(*k.indices(len(self)))]
        k = range(len(self))[k]
        return self.array(k).tolist()

    def array(self, k):
        """Point k's history as a numpy view (no copy)."""
        if self.__dict__.get("_padded") is not None:
            return self._padded[k, :self.iters[k]]
        if self.__dict__.get("_seg") is not None:
            pool, tab, seg = self._seg
            n = int(self.iters[k])
            ids = tab[k, :(n + seg - 1) // seg].astype(np.int64)
            if len(ids) == 1:
                return pool[ids[0] * seg:ids[0] * seg + n]
            return (pool.reshape(-1, seg)[ids].reshape(-1)[:n] if len(ids)
                    else pool[:0])
        return self.flat[self.offsets[k]:self.offsets[k + 1]]


class SegmentedHist:
    """Residual histories of the cluster CG, still on the device: a pool of
    `seg`-entry segments and per point the table of its segments
    (mfb_cg_cluster). `counter` = segments the sweep asked for; when it
    exceeds `cap` some were not stored and the solve must be rerun with
    cap = needed() (the results are deterministic, only histories differ)."""

    def __init__(self, pool, seg_tab, seg, counter, cap):
        self.pool, self.seg_tab, self.seg, self.counter, self.cap = pool, seg_tab, seg, counter, cap

    def needed(self):
        return int(self.counter.item())

    def complete(self):
        return self.needed() <= self.cap

    def to_host(self, iters, n_seg=None):
        """ResidualHistories over host copies of the used segments."""
        import torch
        n_seg = min(self.needed() if n_seg is None else n_seg, self.cap)
        n = n_seg * self.seg
        if 8 * n <= PINNED_HIST_BYTES_MAX:
            # into pinned memory (torch's caching host allocator recycles the
            # block once the caller drops the histories): a pageable copy of a
            # cfg4 batch's histories runs at ~2.4 GB/s
            host = torch.empty(n, dtype=self.pool.dtype, pin_memory=True)
            host.copy_(self.pool[:n])
            flat = host.numpy()
        else:
            # larger than that (a full cfg4 sweep: 9.3 GB): pageable result,
            # moved through a pinned staging buffer, so that results a caller
            # keeps do not pile up as page-locked memory
            flat = np.empty(n, dtype=np.float64)
            step = _HIST_STAGE_DOUBLES
            stage = torch.empty(min(step, n), dtype=self.pool.dtype, pin_memory=True)
            for a in range(0, n, step):
                b = min(a + step, n)
                stage[:b - a].copy_(self.pool[a:b])
                flat[a:b] = stage[:b - a].numpy()
        return ResidualHistories.from_segments(flat, self.seg_tab.cpu().numpy(), iters, self.seg)

    def padded(self, iters, width=None):
        """Device [n_pts, width] tensor of the histories (zeros past each
        point's iterations): the padded layout of the small-interface kernels."""
        import torch
        it = torch.as_tensor(iters, device=self.pool.device).to(torch.int64)
        width = int(it.max().item()) if width is None and it.numel() else int(width or 0)
        width = max(width, 1)
        i = torch.arange(width, device=self.pool.device)
        seg_i = torch.clamp(i // self.seg, max=self.seg_tab.shape[1] - 1)
        sid = self.seg_tab[:, seg_i].to(torch.int64)            # [n_pts, width]
        valid = (i[None, :] < it[:, None]) & (sid >= 0)
        idx = torch.where(valid, sid * self.seg + (i % self.seg)[None, :], 0)
        out = self.pool[idx.clamp(max=max(self.pool.numel() - 1, 0))] if self.pool.numel() \
            else torch.zeros(idx.shape, dtype=torch.float64, device=self.pool.device)
        return torch.where(valid, out, torch.zeros((), dtype=out.dtype, device=out.device))

    def row(self, k, n):
        """Point k's first n entries (host list)."""
        nseg = (int(n) + self.seg - 1) // self.seg
        ids = self.seg_tab[k, :nseg].cpu().numpy()
        out = [self.pool[int(i) * self.seg:(int(i) + 1) * self.seg].cpu().numpy() for i in ids]
        return (np.concatenate(out)[:int(n)] if out else np.zeros(0)).tolist()


def hist_padded(hist, iters):
    """[n_pts, width] device tensor of residual histories from either history
    form a CG launch returns (padded tensor or SegmentedHist)."""
    return hist.padded(iters) if isinstance(hist, SegmentedHist) else hist


def _pack_histories(hist, iters):
    """Device [n_pts, cap] histories -> host ResidualHistories (only the
    first iters[k] entries of row k travel to the host)."""
    import torch
    it_h = np.minimum(iters.cpu().numpy().astype(np.int64), hist.shape[1])
    width = int(it_h.max(initial=0))
    if hist.shape[0] * width * 8 <= (256 << 20):      # small: pack on the host
        h = hist[:, :width].cpu().numpy()
        mask = np.arange(width)[None, :] < it_h[:, None]
        return ResidualHistories(h[mask], it_h)
    it = torch.from_numpy(it_h).to(hist.device)
    mask = torch.arange(width, device=hist.device)[None, :] < it[:, None]
    return ResidualHistories(hist[:, :width][mask].cpu().numpy(), it_h)


def cg_point_order(points, local_idx, local_points, tail=0, width=8):
    """Sweep order and claim chunks of the multi-point CG (mfb_cg_multi).

    The kernel applies a Darcy block once per *distinct* local realization
    among the `width` points a CTA holds, so points that share local
    realizations should sit in the same CTA. Points are sorted (i) longest
    first -- CG iterations grow with the point's largest |coordinate| (cfg4:
    the 64 points at the 15-point rule's extreme node need ~73k iterations,
    the median 20k) --, then (ii) by *reflection family*: the points whose
    local realizations agree up to the sign of each region's local point
    (on a symmetric grid: the 2^m sign combinations of a point with m
    off-centre regions, which visit only two local realizations per such
    region), families of `width` first; a chunk never splits a family. The
    last `tail` points are single-point chunks so the sweep's end stays
    balanced across CTAs. Pure scheduling: the results do not depend on it.

    points [n, n_dims]; local_idx [regions, n]; local_points[r] [N_loc, n_term].
    Returns (order [n] int64, chunk_ptr [n_chunks + 1] int32 into the order).
    """
    n = int(points.shape[0])
    local_idx = np.asarray(local_idx).reshape(-1, n).astype(np.int64)
    key = np.abs(points).max(axis=1) if points.size else np.zeros(n)
    coarse = np.empty_like(local_idx)
    for r in range(local_idx.shape[0]):
        lp = np.round(np.asarray(local_points[r], dtype=np.float64), 9) + 0.0
        lut = {row.tobytes(): i for i, row in enumerate(lp)}
        cls = np.arange(len(lp))
        for i, row in enumerate(lp):
            j = lut.get((-row + 0.0).tobytes())
            if j is not None:
                cls[i] = min(i, j)
        coarse[r] = cls[local_idx[r]]
    o = np.lexsort(tuple(local_idx[::-1]) + tuple(coarse[::-1]) + (-key,))
    sig = np.vstack([key[o][None, :], coarse[:, o].astype(np.float64)])
    new = np.ones(n, dtype=bool)
    new[1:] = (np.diff(sig, axis=1) != 0).any(axis=0)
    fid = np.cumsum(new) - 1
    size = np.minimum(np.bincount(fid)[fid], width)
    o2 = np.lexsort((np.arange(n), fid, -size, -key[o]))
    order, fid = o[o2], fid[o2]
    # chunks: whole families while they fit, cut at `width`; singles in the tail
    n_main = max(0, n - int(tail))
    starts = np.flatnonzero(np.r_[True, fid[1:] != fid[:-1]])
    ends = np.r_[starts[1:], n]
    cptr, fill = [0], 0
    for a, b in zip(starts, ends):
        a, b = int(a), min(int(b), n_main)
        while a < b:
            m = min(b - a, width)
            if fill + m > width:
                cptr.append(cptr[-1] + fill)
                fill = 0
            fill += m
            a += m
            if fill == width:
                cptr.append(cptr[-1] + fill)
                fill = 0
    if fill:
        cptr.append(cptr[-1] + fill)
    cptr = np.concatenate([np.asarray(cptr, dtype=np.int64),
                           np.arange(n_main + 1, n + 1, dtype=np.int64)])
    return order, cptr.astype(np.int32)


def cg_tasks(n_sub, ndof, dof_ptr, dof_map, n_lambda, run=8):
    """Work items of the multi-point CG (mfb_cg_multi): runs of <= `run`
    mortar dofs of one interface with both sides' block rows (an interface's
    dofs are contiguous in both adjacent subdomains' local orders, mortar.py
    sub_dofs), most expensive first, and the strip layout of the packed
    basis pool (mfb_cg_pack): every task side is an 8-row strip of its
    subdomain's block, stored as ceil(ndof / 4) MMA fragments of 32 doubles
    (padded to an even count).

    Returns (tasks [n, 4], sides [n_lambda, 4], strips [m, 4], pk_size
    [n_sub]) int32: task {first dof, strip offset lower, strip offset upper,
    i | (j + 1) << 12 | rows << 24}; per dof {i, row in i, j, row in j}
    (j = -1: none); strip {sid, first row, rows, offset}; packed block size.
    """
    dof_ptr = np.asarray(dof_ptr, dtype=np.int64)
    ndof = np.asarray(ndof, dtype=np.int64)
    sid_of_row = np.repeat(np.arange(n_sub), np.diff(dof_ptr))
    rows = -np.ones((n_lambda, 2), dtype=np.int64)
    for row, d in enumerate(dof_map):
        rows[d, 0 if rows[d, 0] < 0 else 1] = row
    sides = np.full((n_lambda, 4), -1, dtype=np.int64)
    for k in range(2):
        ok = rows[:, k] >= 0
        sid = sid_of_row[rows[ok, k]]
        sides[ok, 2 * k] = sid
        sides[ok, 2 * k + 1] = rows[ok, k] - dof_ptr[sid]
    runs, d = [], 0
    while d < n_lambda:
        i, ai, j, aj = (int(v) for v in sides[d])
        R = 1
        while R < run and d + R < n_lambda:
            i2, a2, j2, b2 = (int(v) for v in sides[d + R])
            if i2 != i or j2 != j or a2 != ai + R or (j >= 0 and b2 != aj + R):
                break
            R += 1
        runs.append((d, i, ai, j, aj, R))
        d += R
    # strips per subdomain in row order
    per_sid = [[] for _ in range(n_sub)]
    for d, i, ai, j, aj, R in runs:
        per_sid[i].append((ai, R))
        if j >= 0:
            per_sid[j].append((aj, R))
    strip_off, strips = {}, []
    pk_size = np.zeros(n_sub, dtype=np.int64)
    for s_ in range(n_sub):
        nt4 = (int(ndof[s_]) + 3) // 4
        w = 32 * (nt4 + (nt4 & 1))       # an even number of fragments per strip (zero-padded)
        for k, (r0, R) in enumerate(sorted(per_sid[s_])):
            strip_off[(s_, r0)] = k * w
            strips.append((s_, r0, R, k * w))
        pk_size[s_] = w * len(per_sid[s_])
    tasks = []
    for d, i, ai, j, aj, R in runs:
        cost = int(ndof[i] + (ndof[j] if j >= 0 else 0))
        tasks.append((-cost, d, strip_off[(i, ai)], strip_off[(j, aj)] if j >= 0 else 0,
                      i | ((j + 1) << 12) | (R << 24)))
    tasks.sort()
    tab = np.array([t[1:] for t in tasks], dtype=np.int32).reshape(-1, 4)
    return (tab, sides.astype(np.int32), np.array(strips, dtype=np.int32).reshape(-1, 4),
            pk_size.astype(np.int32))


def _even_frags(nd):
    nt4 = (int(nd) + 3) // 4
    return nt4 + (nt4 & 1)


def cg_stream_tasks(tab, sides, strips, ndof, region=None, n_warps=16, darcy_groups=2.0):
    """Tasks and strip layout of the streamed multi-point CG (mfb_cg_multi,
    list_cap > 0): two consecutive 8-row tasks of one interface (rows
    consecutive in both subdomains) become one 16-row task whose two strips
    per side share every B operand. Their strips are interleaved in the
    packed pool (pair k of the first strip, then pair k of the second, 128
    doubles per step).

    The kernel's warp w walks tasks w, w + n_warps, ...: the table is laid out
    so that these are the warp's share of a longest-processing-time
    assignment (cost: MMAs of both sides, a Darcy side counted for
    `darcy_groups` local realizations, plus per-pass and per-task overheads),
    its 16-row tasks first; positions without a task hold meta = -1.

    Returns (tab_s [n, 4], strips_s [m, 4]): tasks like cg_tasks' with up to
    16 rows, and the strips with their layout-1 offsets and rows | paired << 8.
    """
    tab = np.asarray(tab, dtype=np.int64)
    strips_s = np.asarray(strips, dtype=np.int64).copy()
    ndof = np.asarray(ndof, dtype=np.int64)
    strip_row = {(int(s_), int(r0)): k for k, (s_, r0, _, _) in enumerate(strips_s)}
    by_d0 = {int(t[0]): t for t in tab}
    out, used = [], set()
    for d0 in sorted(by_d0):
        if d0 in used:
            continue
        _, so_lo, so_up, meta = (int(v) for v in by_d0[d0])
        i, j, R = meta & 0xfff, ((meta >> 12) & 0xfff) - 1, meta >> 24
        ai, aj = int(sides[d0][1]), int(sides[d0][3])
        nxt = by_d0.get(d0 + 8)
        dbl = False
        if R == 8 and nxt is not None:
            m2 = int(nxt[3])
            same = (m2 & 0xfff) == i and ((m2 >> 12) & 0xfff) - 1 == j
            if same and int(sides[d0 + 8][1]) == ai + 8 and \
                    (j < 0 or int(sides[d0 + 8][3]) == aj + 8):
                dbl = True
                used.add(d0 + 8)
                R += m2 >> 24
                for s_, a in ((i, ai), (j, aj)):
                    if s_ < 0:
                        continue
                    ka, kb = strip_row[(s_, a)], strip_row[(s_, a + 8)]
                    assert strips_s[kb, 3] - strips_s[ka, 3] == 32 * _even_frags(ndof[s_])
                    strips_s[kb, 3] = strips_s[ka, 3] + 64
                    strips_s[ka, 2] |= 256
                    strips_s[kb, 2] |= 256
        cost = 4.0
        for s_ in (i, j):
            if s_ >= 0:
                grp = darcy_groups if (region is not None and region[s_] >= 0) else 1.0
                cost += grp * (_even_frags(ndof[s_]) * (2 if dbl else 1) + 2.0)
        out.append((0 if dbl else 1, -cost, d0, so_lo, so_up, i | ((j + 1) << 12) | (R << 24)))
    out.sort(key=lambda t: (t[1], t[0], t[2]))
    load = np.zeros(n_warps)
    mine = [[] for _ in range(n_warps)]
    for t in out:                                   # most expensive first
        w = int(np.argmin(load))
        load[w] -= t[1]
        mine[w].append(t)
    depth = max(len(m) for m in mine)
    tab_s = np.zeros((depth * n_warps, 4), dtype=np.int64)
    tab_s[:, 3] = -1
    for w, m in enumerate(mine):
        for k, t in enumerate(sorted(m)):           # 16-row tasks first
            tab_s[k * n_warps + w] = t[2:]
    return tab_s, strips_s


def _check_basis_cap(sizes_bytes, cap_mb):
    total = sum(sizes_bytes)
    if cap_mb is not None and total > cap_mb * 2 ** 20:
        raise SizeCapError(f"flux basis storage {total / 2 ** 20:.3g} MiB exceeds the "
                           f"cap of {cap_mb:.3g} MiB; raise basis_cap_mb or use method S1")


def _digest(*arrays):
    import hashlib
    h = hashlib.blake2b(digest_size=16)
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str((a.dtype.str, a.shape)).encode())
        h.update(a.view(np.uint8).reshape(-1) if a.size else b"")
    return h.hexdigest()


def _plan_fingerprint(problem, grid):
    """What the resident plan was built from. The reference recomputes
    everything on every call and its problem is a mutable dataclass, so the
    key covers the component objects AND the contents a caller may edit in
    place between calls: the boundary conditions (kind and data per side),
    physics, the mean log-permeability, and the grid's points, weights and
    local tables (hashed). Any change rebuilds the plan."""
    bcs = tuple(sorted((int(s), side, bc.kind, id(bc.value))
                       for s, sides in problem.bcs.items() for side, bc in sides.items()))
    mean = problem.perm.mean
    mean_key = (id(mean), getattr(mean, "kind", None), repr(getattr(mean, "value", None)),
                id(getattr(mean, "func", None)), repr(getattr(mean, "per_region", None)))
    li = list(grid.local_indices) + list(grid.local_points)
    return (id(problem), id(grid), problem.physics, bcs, id(problem.perm),
            tuple(id(r) for r in problem.perm.regions), mean_key,
            id(problem.f_s), id(problem.f_d), id(problem.q_d), id(problem.meshes),
            id(problem.space), id(problem.layout), grid.n_real,
            _digest(grid.points, grid.weights, *li), tuple(grid.local_counts))


def get_plan(problem, grid):
    key = _plan_fingerprint(problem, grid)
    plan = _PLAN_CACHE.pop(key, None)
    if plan is None or plan.problem is not problem or plan.grid is not grid:
        plan = DevicePlan(problem, grid)
    _PLAN_CACHE[key] = plan                 # most recently used last
    while len(_PLAN_CACHE) > PLAN_CACHE_SIZE:
        _PLAN_CACHE.pop(next(iter(_PLAN_CACHE)))
    return plan


class _SweepStatic:
    """Everything a sweep needs that depends only on (problem, grid, method).

    Built once per DevicePlan and kept resident: the system list and its
    offsets, the KL tables, the wave partition of the basis launches with
    their workspaces, the output pools and the moment group tables. A call
    to run_method then only launches kernels and copies results back.

    method "S3" (stochastic MFB, interface.py:349-414): one system per
    (subdomain, local realization of its KL region); Stokes once, frozen at
    the mean field. method "S2" (deterministic MFB, interface.py:317-328):
    one system per (subdomain, global realization) -- Stokes included, with
    the realization's BJS permeability -- and the CG gathers realization k's
    own blocks.
    """

    def __init__(self, plan, keep_fields=True, darcy_kernel="hybrid", method="S3",
                 keep_factors=False, reals=None):
        import torch
        self.darcy_kernel = darcy_kernel
        self.keep_factors = keep_factors
        self.method = method
        pb, grid = plan.problem, plan.grid
        lay = pb.layout
        f64, i32, i64 = torch.float64, torch.int32, torch.int64
        n_real = grid.n_real
        # S2 systems of realizations r0..r1-1 only (Method S1's realization
        # chunks); the K buffer and KL tables still cover every realization
        self.reals = (0, n_real) if reals is None else (int(reals[0]), int(reals[1]))
        if method == "S2":
            r0, r1 = self.reals
            systems = [(s, k) for s in range(plan.n_sub) for k in range(r0, r1)]
            self.n_loc = np.full(plan.n_sub, r1 - r0, dtype=np.int64)
        else:
            systems = plan.s3_systems()
            self.n_loc = plan.n_loc.astype(np.int64).copy()
        self.systems = systems
        nsys = len(systems)
        # (1) KL: K buffer = [K0 (all Darcy cells, mean field) | per-system K].
        # S3: K(sid, loc) per Darcy system. S2: one full K0-layout row per
        # realization (problem.permeability(y_k)); Stokes systems of
        # realization k read their BJS cells from that row.
        koff = np.zeros(nsys, dtype=np.int64)
        first = {}
        for idx, (s, _) in enumerate(systems):
            first.setdefault(s, idx)
        if method == "S2":
            for idx, (s, k) in enumerate(systems):
                koff[idx] = plan.k0_len * (1 + k) + (plan.k0_off[s] if s in plan.k0_off else 0)
            cur = plan.k0_len * (1 + n_real)
        else:
            cur = plan.k0_len
            for idx, (s, l) in enumerate(systems):
                if lay.physics(s) == "darcy":
                    koff[idx] = cur
                    cur += pb.meshes[s].n_cells
        self.koff, self.sys_first = koff, first
        self.K = _scratch("K", max(cur, 1), f64)
        # The sweep's inputs (local-index table, weights, KL tables) live in
        # one device staging buffer (refresh_inputs: one pinned H2D copy);
        # the KL tables are views into it.
        self._plan = plan
        kl_host = [(s, self._kl_tables(plan, s)) for s in plan.darcy]
        sizes = [4 * int(plan.d_local.numel()), 8 * int(plan.d_weights.numel())]
        for _, (phi, mean, xi) in kl_host:
            sizes += [phi.nbytes, mean.nbytes, xi.nbytes]
        offs = np.concatenate([[0], np.cumsum([(b + 15) // 16 * 16 for b in sizes])])
        self._stage_offs = offs
        self._stage_dev = torch.zeros(max(int(offs[-1]), 16), dtype=torch.uint8, device="cuda")

        def view(j, dtype, shape):
            return self._stage_dev[int(offs[j]):int(offs[j]) + sizes[j]].view(dtype).view(shape)

        self.kl = []
        for j, (s, (phi, mean, xi)) in enumerate(kl_host):
            if method == "S2":
                dst, ld = plan.k0_len + plan.k0_off[s], plan.k0_len
            else:
                dst, ld = int(koff[first[s]]), len(mean)
            d_phi = view(2 + 3 * j, f64, phi.shape)
            d_mean = view(3 + 3 * j, f64, mean.shape)
            d_xi = view(4 + 3 * j, f64, xi.shape)
            self.kl.append((s, len(mean), phi.shape[1], d_phi, d_mean, d_xi, int(dst),
                            xi.shape[0] - 1, int(ld)))
        self.refresh_inputs()
        self.kl_h2d_bytes = sum(8 * (t[3].numel() + t[4].numel() + t[5].numel())
                                for t in self.kl)
        # the same tables as one MfbKlTable array: a single batched KL launch
        tabs = (_lib.MfbKlTable * max(len(self.kl), 1))()
        for j, (s_, nc, nt, d_phi, d_mean, d_xi, dst, nrows, ld) in enumerate(self.kl):
            t = tabs[j]
            t.phi, t.mean, t.xi = d_phi.data_ptr(), d_mean.data_ptr(), d_xi.data_ptr()
            t.dst0, t.dst, t.ld = int(plan.k0_off[s_]), int(dst), int(ld)
            if int(nt) > KL_MAX_TERM:
                raise NativeLibraryError(f"KL kernel: {int(nt)} terms in one region exceed "
                                         f"{KL_MAX_TERM}")
            t.n_cells, t.n_term, t.n_rows = int(nc), int(nt), int(nrows)
        self.kl_tab = torch.frombuffer(bytearray(bytes(tabs)), dtype=torch.uint8).to("cuda")
        self.kl_max_rows = max([t[7] for t in self.kl], default=0)
        self.kl_max_cells = max([t[1] for t in self.kl], default=0)
        # CG gather tables: block of subdomain i at point k is loc = table[region_i][k]
        if method == "S2":
            self.d_cg_region = _dev(np.zeros(plan.n_sub, dtype=np.int32), i32)
            self.d_cg_local = _dev(np.arange(n_real, dtype=np.int32)[None, :], i32)
        else:
            self.d_cg_region, self.d_cg_local = plan.d_region, plan.d_local
        # (2) systems: pools and waves
        pats = plan.patterns
        sys_pat = np.array([s for s, _ in systems], dtype=np.int32)
        nd = plan.ndof[sys_pat].astype(np.int64)
        nf = plan.nfield[sys_pat].astype(np.int64)
        boff = np.concatenate([[0], np.cumsum(nd * nd)])
        hoff = np.concatenate([[0], np.cumsum(nd)])
        moff = np.concatenate([[0], np.cumsum(nf * nd)])
        fboff = np.concatenate([[0], np.cumsum(nf)])
        self.keep_fields = keep_fields
        self.blocks = _scratch("blocks", int(boff[-1]), f64)
        self.hbar = _scratch("hbar", int(hoff[-1]), f64)
        self.M = _scratch("M", int(moff[-1]) if keep_fields else 0, f64)
        self.Fb = _scratch("Fb", int(fboff[-1]) if keep_fields else 0, f64)
        self.sys_boff, self.sys_hoff = boff[:-1], hoff[:-1]
        self.sys_moff, self.sys_fboff = moff[:-1], fboff[:-1]
        self.d_pat = _dev(sys_pat, i32)
        self.d_koff = _dev(koff, i64)
        self.d_boff, self.d_hoff = _dev(boff[:-1], i64), _dev(hoff[:-1], i64)
        self.d_moff, self.d_fboff = _dev(moff[:-1], i64), _dev(fboff[:-1], i64)
        phys = [lay.physics(s) for s, _ in systems]
        use_hyb = [ph == "darcy" and self.darcy_kernel == "hybrid" for ph in phys]

        def sub(idx):
            idx = np.asarray(idx, dtype=np.int64)
            return {"idx": idx, "pat": _dev(sys_pat[idx], i32), "koff": _dev(koff[idx], i64),
                    "boff": _dev(boff[:-1][idx], i64), "hoff": _dev(hoff[:-1][idx], i64),
                    "moff": _dev(moff[:-1][idx], i64), "fboff": _dev(fboff[:-1][idx], i64)}

        # generic banded-LU waves (Stokes, or every system when forced)
        self.smem = max(p.smem_doubles for p in pats)
        gen = [i for i in range(nsys) if not use_hyb[i]]
        work_d = {i: pats[systems[i][0]].work_doubles for i in gen}
        x_d = {i: pats[systems[i][0]].x_doubles for i in gen}
        self.waves, wmax, xmax = [], 0, 0
        pos = 0
        while pos < len(gen):
            grp, acc = [], 0
            while pos < len(gen) and (not grp or (acc + 8 * (work_d[gen[pos]] + x_d[gen[pos]])
                                                  <= WORK_BUDGET_BYTES
                                                  and phys[gen[pos]] == phys[grp[0]])):
                acc += 8 * (work_d[gen[pos]] + x_d[gen[pos]])
                grp.append(gen[pos])
                pos += 1
            # keep_factors: every wave gets its own region (the factors and
            # the solutions stay for later solves); else the waves reuse one
            wbase, xbase = (wmax, xmax) if keep_factors else (0, 0)
            woff = wbase + np.concatenate([[0], np.cumsum([work_d[i] for i in grp])])
            xoff = xbase + np.concatenate([[0], np.cumsum([x_d[i] for i in grp])])
            klmax = max(pats[systems[i][0]].kl for i in grp)
            # one panel row per thread when it fits (384 threads keep 170
            # registers per thread, 512 would cap them at 128 and spill)
            nt = 256 if klmax + 16 <= 256 else 384
            if klmax + 16 > 2 * nt:
                raise SizeCapError(f"band half-width {klmax} exceeds the panel kernel's "
                                   f"{2 * nt - 16} (two panel rows per thread)")
            w = sub(grp)
            w["info"] = torch.zeros(len(grp), dtype=i32, device="cuda")
            # CTAs per system: fill the SMs when systems are few (one CTA per SM
            # when the band needs most of the shared memory)
            grpsz = max(1, min(BAND_GROUP_MAX, N_SMS // max(len(grp), 1)))
            w.update(nt=nt, group=grpsz, woff=_dev(woff[:-1], i64), xoff=_dev(xoff[:-1], i64),
                     flops=sum(pats[systems[i][0]].algorithmic_flops for i in grp))
            self.waves.append(w)
            wmax, xmax = max(wmax, int(woff[-1])), max(xmax, int(xoff[-1]))
        # hybrid (SPD condensation) waves for Darcy systems, grouped by panel width
        hyb = [i for i in range(nsys) if use_hyb[i]]
        self.hwaves = []
        lmax = hxmax = 0
        for panel in (16, 8):
            idxs = [i for i in hyb if plan.hyb_panel[systems[i][0]] == panel]
            pos = 0
            while pos < len(idxs):
                grp, acc = [], 0
                while pos < len(idxs):
                    h = plan.hyb[systems[idxs[pos]][0]]
                    _, _, _, ld, xd = h.layout_for(panel)
                    cost = 8 * (ld + xd) if keep_fields else 0
                    if grp and acc + cost > WORK_BUDGET_BYTES:
                        break
                    acc += cost
                    grp.append(idxs[pos])
                    pos += 1
                lays = [plan.hyb[systems[i][0]].layout_for(panel) for i in grp]
                loff = np.concatenate([[0], np.cumsum([l[3] for l in lays])])
                hxoff = np.concatenate([[0], np.cumsum([l[4] for l in lays])])
                w = sub(grp)
                w["info"] = torch.zeros(len(grp), dtype=i32, device="cuda")
                wmax_ = max(plan.hyb[systems[i][0]].w for i in grp)
                w.update(panel=panel, rl=-(-(wmax_ + panel) // 32), smem_c=max(l[1] for l in lays),
                         smem_b=max(l[2] for l in lays), loff=_dev(loff[:-1], i64),
                         xoff=_dev(hxoff[:-1], i64),
                         flops=sum(plan.hyb[systems[i][0]].algorithmic_flops for i in grp),
                         survey_flops=sum(pats[systems[i][0]].algorithmic_flops for i in grp))
                self.hwaves.append(w)
                lmax, hxmax = max(lmax, int(loff[-1])), max(hxmax, int(hxoff[-1]))
        self.work = _scratch("work", max(wmax, 1), f64)
        # per system: group-barrier counter and panel-ready counter (mfb_band.cu)
        self.bar = torch.zeros(2 * max(len(systems), 1), dtype=torch.int32, device="cuda")
        self.X = _scratch("X", max(xmax, 1), f64)
        self.Lstore = _scratch("Lstore", max(lmax, 1) if keep_fields else 1, f64)
        self.HX = _scratch("HX", max(hxmax, 1) if keep_fields else 1, f64)
        self.blk_base = np.array([boff[first[s]] for s in range(plan.n_sub)], dtype=np.int64)
        self.h_base = np.array([hoff[first[s]] for s in range(plan.n_sub)], dtype=np.int64)
        self.d_blk, self.d_h = _dev(self.blk_base, i64), _dev(self.h_base, i64)
        # (4) moment groups = systems; members from the region local-index tables
        members, gptr, order_cache = [], [0], {}
        for s, l in systems:
            r = plan.region[s]
            if method == "S2":                  # one realization per system
                mem = np.array([l])
            elif r < 0:
                mem = np.arange(grid.n_real)
            else:
                if r not in order_cache:
                    li = grid.local_indices[r]
                    order = np.argsort(li, kind="stable")
                    bounds = np.searchsorted(li[order], np.arange(grid.local_counts[r] + 1))
                    order_cache[r] = (order, bounds)
                order, bounds = order_cache[r]
                mem = order[bounds[l]:bounds[l + 1]]
            members.append(mem)
            gptr.append(gptr[-1] + len(mem))
        voff = np.concatenate([[0], np.cumsum(nd)])
        coff = np.concatenate([[0], np.cumsum(nd * nd)])
        self._members, self._voff, self._coff = members, voff, coff
        self._moff, self._fboff = moff, fboff
        self.nv, self.nc = int(voff[-1]), int(coff[-1])
        self.out_off = np.concatenate([[0], np.cumsum(plan.nfield.astype(np.int64))])
        self._mtab = {}
        self._wave_cache = {}
        self.wtot = float(np.sum(grid.weights))


    def moment_table(self, sids):
        """Device group tables restricted to the systems of `sids` (cached)."""
        key = tuple(sids)
        tab = self._mtab.get(key)
        if tab is not None:
            return tab
        import torch
        plan = self._plan
        i32, i64 = torch.int32, torch.int64
        sel = [i for i, (s, _) in enumerate(self.systems) if s in set(sids)]
        gptr = np.concatenate([[0], np.cumsum([len(self._members[i]) for i in sel])])
        mem = np.concatenate([self._members[i] for i in sel]) if sel else np.zeros(1, int)
        sys_pat = np.array([self.systems[i][0] for i in sel], dtype=np.int32)
        sgptr, cur = [0], 0
        for s in sids:
            cur += sum(1 for i in sel if self.systems[i][0] == s)
            sgptr.append(cur)
        nf = plan.nfield[list(sids)].astype(np.int64)
        out_off = np.concatenate([[0], np.cumsum(nf)])
        keys, kstart, kshape = [], [], []
        for j, s in enumerate(sids):
            for name, start, shape in plan.patterns[s].field_layout:
                keys.append(f"{s}:{name}")
                kstart.append(int(out_off[j] + start))
                kshape.append(tuple(shape))
        tab = {"n": len(sel), "pat": _dev(sys_pat, i32), "gptr": _dev(gptr, i32),
               "keys": keys, "key_start": np.array(kstart, dtype=np.int64), "key_shape": kshape,
               "key_slices": [(k, a, a + int(np.prod(sh)), sh)
                              for k, a, sh in zip(keys, kstart, kshape)],
               "mem": _dev(mem, i32), "voff": _dev(self._voff[:-1][sel], i64),
               "coff": _dev(self._coff[:-1][sel], i64),
               "moff": _dev(self._moff[:-1][sel], i64),
               "fboff": _dev(self._fboff[:-1][sel], i64),
               "sgptr": _dev(np.array(sgptr), i32), "nfield": _dev(nf.astype(np.int32), i32),
               "out_off": out_off, "d_outoff": _dev(out_off[:-1], i64), "sids": list(sids)}
        self._mtab[key] = tab
        return tab

    def waves_for(self, sids):
        """The basis waves restricted to the systems of `sids` (cached)."""
        if sids is None:
            return self.waves, self.hwaves
        key = tuple(sorted(sids))
        if key not in self._wave_cache:
            import torch
            keep = set(key)
            out = []
            for wl in (self.waves, self.hwaves):
                sub = []
                for w in wl:
                    m = np.array([self.systems[i][0] in keep for i in w["idx"]])
                    if not m.any():
                        continue
                    nw = {}
                    for k, v in w.items():
                        if isinstance(v, torch.Tensor) and v.numel() == len(w["idx"]):
                            nw[k] = v[torch.as_tensor(np.nonzero(m)[0], device=v.device)]
                        elif k == "idx":
                            nw[k] = v[m]
                        else:
                            nw[k] = v
                    sub.append(nw)
                out.append(sub)
            self._wave_cache[key] = tuple(out)
        return self._wave_cache[key]

    def _kl_tables(self, plan, s):
        """Phi, mean and the xi rows (row 0 = the mean field) of Darcy sid s
        (host arrays, evaluated once per plan like the rest of the setup)."""
        cache = self.__dict__.setdefault("_kl_host", {})
        if s not in cache:
            cache[s] = self._kl_tables_eval(plan, s)
        return cache[s]

    def _kl_tables_eval(self, plan, s):
        pb, grid = plan.problem, plan.grid
        r = pb.layout.blocks[s].kl_region
        c = pb.meshes[s].centroids
        phi, mean = mode_table(pb.perm, r, c[:, 0], c[:, 1])
        nt = phi.shape[1]
        pts = grid.local_points[r][:, :nt]
        if self.method == "S2":        # realization k's region coordinates
            pts = pts[np.asarray(grid.local_indices[r])]
        xi = np.zeros((1 + len(pts), nt))
        xi[1:] = pts
        return phi, mean, xi

    def side_stream(self):
        """Second stream for the banded (Stokes) waves of build_bases."""
        if getattr(self, "_side", None) is None:
            import torch
            # high priority: the work put here (the Stokes systems) is the
            # critical path, its CTAs are dispatched ahead of the other stream's
            self._side = torch.cuda.Stream(priority=-1)
        return self._side

    def refresh_inputs(self):
        """Re-upload the sweep's inputs from the host -- local-index tables,
        collocation weights and the KL tables (Phi, mean, local points) -- in
        ONE pinned host->device copy into the staging buffer the KL kernels
        read; the plan's local-index table and weights are copied out of it
        on the device. Returns the bytes transferred."""
        import torch
        plan, grid = self._plan, self._plan.grid
        li = np.stack(grid.local_indices).astype(np.int32) if grid.local_indices else \
            np.zeros((1, grid.n_real), dtype=np.int32)
        pieces = [li, np.ascontiguousarray(grid.weights)]
        offs = self._stage_offs
        # the KL tables (evaluated once per plan, _kl_tables) as one byte image
        kl_img = getattr(self, "_kl_image", None)
        if kl_img is None:
            kl_img = np.zeros(int(offs[-1]) - int(offs[2]), dtype=np.uint8)
            j = 2
            for s_, *_ in self.kl:
                for h in self._kl_tables(plan, s_):
                    b = np.ascontiguousarray(h).view(np.uint8).ravel()
                    a = int(offs[j]) - int(offs[2])
                    kl_img[a:a + b.nbytes] = b
                    j += 1
            self._kl_image = kl_img
        host = getattr(self, "_stage_host", None)
        if host is None:
            host = self._stage_host = torch.empty(self._stage_dev.numel(), dtype=torch.uint8,
                                                  pin_memory=True)
        ev = getattr(self, "_stage_ev", None)
        if ev is not None:
            ev.synchronize()                     # the previous upload left the pinned buffer
        hv = host.numpy()
        for h, o in zip(pieces, offs):
            b = np.ascontiguousarray(h)
            hv[int(o):int(o) + b.nbytes] = b.view(np.uint8).ravel()
        hv[int(offs[2]):int(offs[2]) + kl_img.nbytes] = kl_img
        self._stage_dev.copy_(host, non_blocking=True)
        self._stage_ev = torch.cuda.Event()
        self._stage_ev.record()
        n0, n1 = int(plan.d_local.numel()), int(plan.d_weights.numel())
        plan.d_local.view(-1).copy_(self._stage_dev[:4 * n0].view(torch.int32))
        plan.d_weights.copy_(
            self._stage_dev[int(offs[1]):int(offs[1]) + 8 * n1].view(torch.float64))
        return int(offs[-1])


class SweepEngine:
    """Device work of one S3 or S2 sweep; methods map 1:1 onto the C ABI calls."""

    def __init__(self, plan, stream=None, keep_fields=True, darcy_kernel="hybrid", method="S3",
                 keep_factors=False, reals=None):
        import torch
        self.torch = torch
        self.plan = plan
        self.method = method
        self.L = _lib.lib()
        self.st = plan.sweep_static(keep_fields, darcy_kernel, method, keep_factors, reals)
        self.stream = torch.cuda.current_stream() if stream is None else stream
        self.sp = ctypes.c_void_p(self.stream.cuda_stream)
        self.launches = 0            # kernels launched through the C ABI
        self.timing = False          # record CUDA events around the basis solves and CG
        self.wave_timing = False     # events around every basis wave (run_method: wall_seconds)
        self.wave_events = []
        self.solve_events = []
        self.bases_events = []
        self.cg_events = []
        self.solve_flops = []

    def __getattr__(self, name):     # pools live in the static state
        return getattr(self.__dict__["st"], name)

    def _ev(self, stream=None):
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(self.stream if stream is None else stream)
        return ev

    # ------------------------------------------------------------ (1) KL --
    def kl_fields(self):
        """K for every (Darcy sid, loc) system plus the mean-field K0 buffer."""
        _claim(self.st, "K")
        st, plan = self.st, self.plan
        K = st.K
        if st.kl:
            self.launches += 1
            _lib.check(self.L.mfb_kl_realize_batched(
                len(st.kl), _ptr(st.kl_tab), st.kl_max_rows, st.kl_max_cells, _ptr(K), self.sp),
                "mfb_kl_realize_batched")
        return K

    # ------------------------------------------------------- (2) bases ----
    def build_bases(self, sids=None):
        """Every (subdomain, realization) system of the sweep. The banded
        (Stokes) waves run on a second stream, concurrently with the Darcy
        condensation on the engine's stream: the cooperative Stokes solve is
        latency bound and leaves SMs free. Both write disjoint pool slices;
        the engine's stream waits for the side stream before returning."""
        torch = self.torch
        st, plan = self.st, self.plan
        _check_owner(st, "K")
        _claim(st, "blocks", "hbar", "M", "Fb", "work", "X", "Lstore", "HX")
        waves, hwaves = st.waves_for(sids)
        self._last_waves = list(waves) + list(hwaves)
        if self.timing:
            eb0 = self._ev()
        side = None
        if waves and hwaves:
            side = st.side_stream()
            side.wait_stream(self.stream)           # K from the KL launches
        bs = side if side is not None else self.stream
        sp_b = ctypes.c_void_p(bs.cuda_stream)
        self.wave_events = []
        for w in waves:                         # generic banded LU (Stokes)
            cnt = len(w["idx"])
            if self.wave_timing:
                w0 = self._ev(bs)
            if self.timing:
                e0 = self._ev(bs)
            _lib.check(self.L.mfb_systems_solve(
                _ptr(plan.pat_dev), cnt, _ptr(w["pat"]), _ptr(st.K), _ptr(w["koff"]),
                _ptr(st.work), _ptr(w["woff"]), _ptr(st.X), _ptr(w["xoff"]), _ptr(w["info"]),
                w["nt"], st.smem, w["group"], _ptr(st.bar), int(st.keep_factors), sp_b),
                "mfb_systems_solve")
            if self.timing:
                self.solve_events.append(("band", e0, self._ev(bs), w["flops"], w["flops"]))
            self.launches += 2
            _lib.check(self.L.mfb_systems_extract(
                _ptr(plan.pat_dev), cnt, _ptr(w["pat"]), _ptr(st.X), _ptr(w["xoff"]),
                _ptr(st.blocks), _ptr(w["boff"]), _ptr(st.hbar), _ptr(w["hoff"]),
                _ptr(st.M) if st.keep_fields else None, _ptr(w["moff"]),
                _ptr(st.Fb) if st.keep_fields else None, _ptr(w["fboff"]), sp_b),
                "mfb_systems_extract")
            if SYMMETRIZE_BAND_BLOCKS and not st.keep_factors:
                # the banded LU leaves ~1e-12 of asymmetry in a block that is
                # symmetric (the reference's: 3e-13); the unpreconditioned CG
                # pays ~10% more iterations for it (mfb.h)
                self.launches += 1
                _lib.check(self.L.mfb_blocks_symmetrize(
                    _ptr(plan.pat_dev), cnt, _ptr(w["pat"]), _ptr(st.blocks), _ptr(w["boff"]),
                    sp_b), "mfb_blocks_symmetrize")
            if self.wave_timing:
                self.wave_events.append((w, w0, self._ev(bs)))
        for w in hwaves:                        # hybridised Darcy condensation
            cnt = len(w["idx"])
            keep = st.keep_fields
            if self.wave_timing:
                w0 = self._ev()
            if self.timing:
                e0 = self._ev()
            _lib.check(self.L.mfb_darcy_condense(
                _ptr(plan.hyb_dev), cnt, _ptr(w["pat"]), _ptr(st.K), _ptr(w["koff"]),
                _ptr(st.blocks), _ptr(w["boff"]), _ptr(st.hbar), _ptr(w["hoff"]),
                _ptr(st.Lstore) if keep else None, _ptr(w["loff"]), _ptr(w["info"]),
                w["panel"] | (w["rl"] << 8), w["smem_c"], self.sp), "mfb_darcy_condense")
            if self.timing:
                self.solve_events.append(("hybrid", e0, self._ev(), w["flops"],
                                          w["survey_flops"]))
            self.launches += 1
            if keep:
                self.launches += 2
                _lib.check(self.L.mfb_darcy_backsolve(
                    _ptr(plan.hyb_dev), cnt, _ptr(w["pat"]), _ptr(st.Lstore), _ptr(w["loff"]),
                    _ptr(st.HX), _ptr(w["xoff"]), w["panel"], w["smem_b"], self.sp),
                    "mfb_darcy_backsolve")
                _lib.check(self.L.mfb_darcy_recover(
                    _ptr(plan.hyb_dev), cnt, _ptr(w["pat"]), _ptr(st.K), _ptr(w["koff"]),
                    _ptr(st.HX), _ptr(w["xoff"]), _ptr(st.M), _ptr(w["moff"]), _ptr(st.Fb),
                    _ptr(w["fboff"]), self.sp), "mfb_darcy_recover")
            if self.wave_timing:
                self.wave_events.append((w, w0, self._ev()))
        if side is not None:
            self.stream.wait_stream(side)
            # the side stream's allocations-in-flight: none (all buffers are
            # the static pools), so no record_stream bookkeeping is needed
        if self.timing:                 # wall time of the whole basis phase
            self.bases_events.append((eb0, self._ev()))

    def check_info(self):
        info = np.zeros(len(self.st.systems), dtype=np.int64)
        for w in getattr(self, "_last_waves", self.st.waves + self.st.hwaves):
            info[w["idx"]] = w["info"].cpu().numpy()
        bad = np.nonzero(info != 0)[0]
        if len(bad):
            s, l = self.st.systems[bad[0]]
            raise SingularOperatorError(
                f"subdomain {s} (local realization {l}): singular system "
                f"(device info {int(info[bad[0]])})")

    def subdomain_seconds(self, n_sub):
        """Device time of the basis phase per subdomain (after a sync): every
        wave's measured time (CUDA events around its launches: assembly,
        factorization, basis columns, bar solve, field responses) shared
        equally among its systems -- a wave holds systems of one pattern --
        and summed per subdomain. The reference accumulates the wall time of
        the same per-subdomain work (interface.py:142-154); the waves of the
        two streams overlap, so the sum can exceed the phase's wall time."""
        sec = np.zeros(n_sub)
        for w, e0, e1 in self.wave_events:
            idx = np.asarray(w["idx"]).astype(np.int64).reshape(-1)
            if len(idx) == 0:
                continue
            sids = np.array([self.st.systems[int(i)][0] for i in idx], dtype=np.int64)
            np.add.at(sec, sids, e0.elapsed_time(e1) / 1e3 / len(idx))
        return sec

    # ---------------------------------------------------------- (3) CG ----
    def solve_points(self, tol, max_iter, k0=0, n_pts=None, hist_cap=None, keep_g=False,
                     kernel="auto", cluster_shape=None, hist_segments=None, check_hist=False,
                     local_override=None):
        """CG over points k0..k0+n_pts-1. kernel: "auto" (multi-point when the
        blocks exceed shared memory and the points fill the GPU, else one CTA
        per point with register-resident block rows when they fit), "cta"
        (one CTA per point), "staged" (one CTA per point, blocks staged in
        shared memory), "multi" (8 points per CTA, forced, for tests) or
        "cluster" (NP points per thread-block cluster, forced; the "auto"
        choice is "multi" for large interfaces). The multi and cluster kernels
        return their residual histories as a SegmentedHist, the others as
        [n_pts, hist_cap]."""
        torch, plan, st = self.torch, self.plan, self.st
        _check_owner(st, "blocks", "hbar")
        n_real = plan.grid.n_real
        cg_local = st.d_cg_local
        if local_override is not None:
            # points 0..n-1 of a caller-built local-index table [regions, n]
            # (distributed.py: a rank's interleaved points)
            cg_local = local_override
            n_real, k0 = int(local_override.shape[1]), 0
        n_pts = n_real - k0 if n_pts is None else n_pts
        nl = plan.n_lambda
        hist_cap = max_iter if hist_cap is None else hist_cap
        lam = torch.empty((n_pts, nl), dtype=torch.float64, device="cuda")
        iters = torch.empty(n_pts, dtype=torch.int32, device="cuda")
        status = torch.empty(n_pts, dtype=torch.int32, device="cuda")
        g = torch.empty((n_pts, nl), dtype=torch.float64, device="cuda") if keep_g else None
        self.launches += 1
        if self.timing:
            e0 = self._ev()
        ct = None
        if kernel == "cluster":
            ct = self._cluster_tables(n_pts, force=True, shape=cluster_shape)
            if ct is None:
                raise NativeLibraryError("no cluster shape fits this interface")
        mt = None
        if ct is None and kernel not in ("cta", "staged"):
            mt = self._multi_tables(n_pts, force=kernel == "multi")
        if ct is not None or mt is not None:
            # the large-interface kernels keep residual histories in segments
            # (device memory ~ the iterations run, not n_pts x max_iter)
            mt = self._pack_tables() if mt is None else mt
            # streamed S p (pass lists in shared memory) when they fit
            stream = ct is None and MULTI_STREAM and mt["list_cap"] > 0
            self._repack(mt, layout=1 if stream else 0)
            # Sweep order (cg_point_order): longest points first, and points
            # that share local realizations next to each other, claimed by a
            # CTA in chunks. Every point's arithmetic is independent of its
            # slot: the outputs are the same bits, scattered back to point
            # order below.
            order, chunks = None, None
            if (ct is None and local_override is None and n_pts >= 4 * N_SMS
                    and plan.grid.n_dims and st.method != "S2" and MULTI_CHUNKS):
                o, cptr = cg_point_order(
                    np.asarray(plan.grid.points[k0:k0 + n_pts]),
                    plan.host.local[:, k0:k0 + n_pts], plan.grid.local_points,
                    tail=mt["n_cta"] * 8 if MULTI_TAIL is None else MULTI_TAIL)
                order = torch.as_tensor(o, device="cuda")
                chunks = torch.as_tensor(cptr, dtype=torch.int32, device="cuda")
            elif local_override is None and n_pts >= 4 * N_SMS and plan.grid.n_dims:
                key = np.abs(np.asarray(plan.grid.points[k0:k0 + n_pts])).max(axis=1)
                o = np.argsort(-key, kind="stable")
                if np.any(o != np.arange(n_pts)):
                    order = torch.as_tensor(o, device="cuda")
            if order is not None:
                cg_local = st.d_cg_local[:, k0 + order].contiguous()
                n_real, k0 = n_pts, 0
            seg = HIST_SEG
            max_segs = (int(max_iter) + seg - 1) // seg
            # The segment pool of the last solve is reused when nobody holds
            # its histories any more (allocating several GB per call costs
            # ~0.4 s with expandable segments).
            pool = _HIST_POOL.pop("pool", None)      # (one pool for every plan)
            if pool is not None and sys.getrefcount(pool) > 2:
                pool = None
            cap = hist_segments
            if cap is None and pool is not None and pool.numel() >= n_pts * seg:
                cap = pool.numel() // seg
            elif cap is None:
                pool = None
                free = torch.cuda.mem_get_info()[0]
                # room for a mean of 64 segments (65k iterations) per point,
                # within an eighth of free memory; an overflow reruns exactly
                cap = int(min(n_pts * min(max_segs, 64), max(free // 8, 1 << 28) // (8 * seg)))
            counter = ct["seg_counter"] if ct is not None else mt["seg_counter"]
            while True:
                if pool is None or pool.numel() != int(cap) * seg:
                    pool = None
                    pool = torch.empty(int(cap) * seg, dtype=torch.float64, device="cuda")
                _HIST_POOL["pool"] = pool
                seg_tab = torch.empty((n_pts, max_segs), dtype=torch.int32, device="cuda")
                self.launches += 1
                if ct is not None:
                    C, NP = ct["C"], ct["NP"]
                    self.cg_kernel_name = (f"cg_cluster_kernel<{NP}> ({NP} points per cluster "
                                           f"of {C} CTAs, FP64 mma.m8n8k4, vectors on chip)")
                    _lib.check(self.L.mfb_cg_cluster(
                        nl, C, NP, _ptr(ct["d_hdr"]), _ptr(ct["d_tab"]), ct["n_own_max"],
                        ct["n_used_max"], ct["n_cut_max"], ct["n_cm_max"], ct["n_unit_max"],
                        ct["n_strip_max"], ct["flags"], ct["smem"], _ptr(plan.d_ndof),
                        _ptr(st.d_cg_region), int(st.d_cg_local.shape[0]), _ptr(st.d_h),
                        _ptr(cg_local), n_real, _ptr(st.hbar), _ptr(mt["sides"]),
                        _ptr(mt["packed"]), k0, n_pts, float(tol), int(max_iter), _ptr(lam),
                        _ptr(iters), _ptr(status), _ptr(g) if keep_g else None, _ptr(ct["xs"]),
                        _ptr(ct["rs"]), _ptr(ct["ss"]), ct["n_clusters"], _ptr(mt["counter"]),
                        _ptr(pool), seg, int(cap), _ptr(seg_tab), max_segs, _ptr(counter),
                        self.sp), "mfb_cg_cluster")
                else:
                    self.cg_kernel_name = ("cg_multi_kernel (8 points per CTA on FP64 mma.m8n8k4"
                                       + (", S p streamed over pass lists)" if stream else ")"))
                    _lib.check(self.L.mfb_cg_multi(
                        nl, plan.n_sub, int(plan.dof_ptr[-1]), _ptr(plan.d_ndof),
                        _ptr(plan.d_dof_ptr), _ptr(plan.d_dof_map), _ptr(st.d_cg_region),
                        int(st.d_cg_local.shape[0]), _ptr(st.d_blk), _ptr(st.d_h),
                        _ptr(cg_local), n_real, _ptr(st.blocks), _ptr(st.hbar), k0, n_pts,
                        float(tol), int(max_iter), _ptr(lam), _ptr(iters), _ptr(status),
                        _ptr(pool), seg, _ptr(g) if keep_g else None, _ptr(mt["tasks"]),
                        mt["n_tasks_s" if stream else "n_tasks"], _ptr(mt["sides"]),
                        _ptr(mt["packed"]),
                        _ptr(mt["pk_base"]), _ptr(mt["pk_size"]), mt["n_cta"],
                        _ptr(mt["scratch"]), _ptr(mt["counter"]), _ptr(seg_tab), max_segs,
                        int(cap), _ptr(counter), _ptr(mt["trec_s" if stream else "trec"]),
                        _ptr(chunks) if chunks is not None else None,
                        int(chunks.numel()) - 1 if chunks is not None else 0,
                        mt["list_cap"] if stream else 0,
                        _ptr(mt["dm_pairs" if stream else "dm_rows"]),
                        int(mt["dm_pairs" if stream else "dm_rows"].numel()), self.sp),
                        "mfb_cg_multi")
                hist = SegmentedHist(pool, seg_tab, seg, counter, cap)
                if not check_hist or hist.complete():   # complete() syncs the stream
                    break
                cap = hist.needed()          # rerun once with the exact pool size
            if order is not None:            # back to point order
                def unperm(t):
                    out = torch.empty_like(t)
                    out[order] = t
                    return out
                lam, iters, status = unperm(lam), unperm(iters), unperm(status)
                g = unperm(g) if g is not None else None
                hist.seg_tab = unperm(hist.seg_tab)
            if self.timing:
                self.cg_events.append((e0, self._ev(), n_pts))
            return lam, iters, status, hist, g
        hist = torch.empty((n_pts, max(hist_cap, 1)), dtype=torch.float64, device="cuda")
        # block rows in registers when every ndof is a multiple of 4 (the
        # accumulation order then equals the staged kernel's)
        reg_ndof = int(plan.ndof.max()) if (kernel != "staged" and len(plan.ndof)
                                             and not np.any(plan.ndof % 4)) else 0
        self.cg_kernel_name = (
            "cg_pair_kernel (one CTA per point, block rows in registers)"
            if 0 < reg_ndof <= 32 and 2 * nl <= 608 else
            "cg_kernel (one CTA per point, blocks staged in shared memory or read from L2)")
        if st.blocks.numel() >= 2 ** 31:
            raise NativeLibraryError("the one-CTA-per-point CG addresses the basis pool with "
                                     "32-bit offsets: pool of 2^31 doubles or more")
        _lib.check(self.L.mfb_cg_batched(
            nl, plan.n_sub, _ptr(plan.d_ndof), _ptr(plan.d_dof_ptr), _ptr(plan.d_dof_map),
            _ptr(st.d_cg_region), _ptr(st.d_blk), _ptr(st.d_h), _ptr(cg_local), n_real,
            _ptr(st.blocks), _ptr(st.hbar), k0, n_pts, float(tol), int(max_iter),
            _ptr(lam), _ptr(iters), _ptr(status), _ptr(hist), max(hist_cap, 1),
            _ptr(g) if keep_g else None, int(np.sum(plan.ndof.astype(np.int64) ** 2)),
            reg_ndof, self.sp), "mfb_cg_batched")
        if self.timing:
            self.cg_events.append((e0, self._ev(), n_pts))
        return lam, iters, status, hist, g

    def _pack_tables(self):
        """Task / strip tables of the multi-point CG kernels and the packed
        basis pool (cached on the static state; the pool is repacked by
        mfb_cg_pack on every solve, after the bases)."""
        torch, st, plan = self.torch, self.st, self.plan
        mt = getattr(st, "_multi", None)
        if mt is None:
            nd = plan.ndof.astype(np.int64)
            nl = int(plan.n_lambda)
            tab, sides, strips, pk_size = cg_tasks(plan.n_sub, nd, plan.dof_ptr, plan.dof_map,
                                                   nl)
            n_loc = st.n_loc.astype(np.int64)
            pk_base = np.concatenate([[0], np.cumsum(pk_size.astype(np.int64) * n_loc)])
            if pk_base[-1] >= 2 ** 31:
                raise NativeLibraryError("packed basis pool exceeds 2^31 doubles")
            # per task record (mfb_cg_multi): the run, then per side (nd |
            # (CG region + 1) << 16, dof_ptr) and (strip base, block size)
            creg = (np.zeros(plan.n_sub, dtype=np.int64) if self.st.method == "S2"
                    else plan.region.astype(np.int64))
            trec = np.zeros((len(tab), 12), dtype=np.int64)
            for t, (d0, so_lo, so_up, meta) in enumerate(tab.astype(np.int64)):
                i, j = meta & 0xfff, ((meta >> 12) & 0xfff) - 1
                trec[t, :4] = (d0, so_lo, so_up, meta)
                trec[t, 4] = nd[i] | ((creg[i] + 1) << 16)
                trec[t, 6] = plan.dof_ptr[i]
                trec[t, 8] = pk_base[i] + so_lo
                trec[t, 10] = pk_size[i]
                if j >= 0:
                    trec[t, 5] = nd[j] | ((creg[j] + 1) << 16)
                    trec[t, 7] = plan.dof_ptr[j]
                    trec[t, 9] = pk_base[j] + so_up
                    trec[t, 11] = pk_size[j]
            # dof lists as p offsets (mfb.h: the slot halves of every other dof
            # pair exchanged), row order for the task loop
            dmap = np.asarray(plan.dof_map, dtype=np.int64)
            swz = dmap * 8 + ((dmap & 2) << 1)
            dm_rows = np.concatenate([swz, np.zeros(8, dtype=np.int64)])
            # streamed S p (mfb_cg_multi list_cap > 0): 16-row tasks where an
            # interface allows, their strips interleaved; dof lists padded to 8
            # columns per subdomain and pair-interleaved
            tab_s, strips_s = cg_stream_tasks(tab, sides, strips, nd, creg)
            ndp = (nd + 7) // 8 * 8
            dmo2 = np.concatenate([[0], np.cumsum(ndp)])
            dm_pairs = np.zeros(int(dmo2[-1]), dtype=np.int64)
            for s_ in range(plan.n_sub):
                c = np.arange(int(nd[s_]))
                dm_pairs[dmo2[s_] + (c & ~7) + 2 * (c & 3) + ((c >> 2) & 1)] = \
                    swz[plan.dof_ptr[s_]:plan.dof_ptr[s_] + nd[s_]]
            # per warp (task t on warp t mod 16) one list entry per pass -- at
            # most 8 local-realization groups per Darcy side -- plus a record
            # per task and the end mark
            trec_s = np.zeros((len(tab_s), 12), dtype=np.int64)
            per_task = np.ones(len(tab_s), dtype=np.int64)
            for t, (d0, so_lo, so_up, meta) in enumerate(tab_s):
                trec_s[t, :4] = (d0, so_lo, so_up, meta)
                if meta < 0:                        # no task at this position
                    per_task[t] = 0
                    continue
                i, j = meta & 0xfff, ((meta >> 12) & 0xfff) - 1
                trec_s[t, 4] = nd[i] | ((creg[i] + 1) << 16)
                trec_s[t, 6] = dmo2[i]
                trec_s[t, 8] = pk_base[i] + so_lo
                trec_s[t, 10] = pk_size[i]
                per_task[t] += 8 if creg[i] >= 0 else 1
                if j >= 0:
                    trec_s[t, 5] = nd[j] | ((creg[j] + 1) << 16)
                    trec_s[t, 7] = dmo2[j]
                    trec_s[t, 9] = pk_base[j] + so_up
                    trec_s[t, 11] = pk_size[j]
                    per_task[t] += 8 if creg[j] >= 0 else 1
            list_cap = max(int(per_task[w::16].sum()) for w in range(16)) + 1
            if (int(nd.max()) > 248 or len(dm_pairs) >= 65536
                    or self.L.mfb_cg_multi_smem(nl, len(dm_pairs), list_cap) + 8192 > 227 * 1024):
                list_cap = 0
            mt = {"tasks": _dev(tab.ravel(), torch.int32), "n_tasks": int(len(tab)),
                  "list_cap": list_cap, "n_tasks_s": int(len(tab_s)),
                  "strips_s": _dev(strips_s.ravel(), torch.int32),
                  "trec_s": _dev(trec_s.ravel().astype(np.int32), torch.int32),
                  "dm_rows": _dev(dm_rows, torch.int32), "dm_pairs": _dev(dm_pairs, torch.int32),
                  "trec": _dev(trec.ravel().astype(np.int32), torch.int32),
                  "sides": _dev(sides.ravel(), torch.int32),
                  "strips": _dev(strips.ravel(), torch.int32), "n_strips": int(len(strips)),
                  "pk_size": _dev(pk_size, torch.int32), "pk_base": _dev(pk_base[:-1], torch.int64),
                  "n_loc": _dev(n_loc.astype(np.int32), torch.int32),
                  "max_loc": int(n_loc.max()),
                  "packed": torch.empty(int(pk_base[-1]), dtype=torch.float64, device="cuda"),
                  "counter": torch.zeros(1, dtype=torch.int32, device="cuda"),
                  "seg_counter": torch.zeros(1, dtype=torch.int32, device="cuda"),
                  "host": {"tasks": tab, "sides": sides, "strips": strips, "pk_size": pk_size,
                           "pk_base": pk_base[:-1]}}
            st._multi = mt
        return mt

    def _repack(self, mt, layout=0):
        plan, st = self.plan, self.st
        self.launches += 1
        _lib.check(self.L.mfb_cg_pack(
            mt["n_strips"], _ptr(mt["strips_s" if layout else "strips"]), _ptr(plan.d_ndof),
            _ptr(mt["n_loc"]),
            mt["max_loc"], _ptr(st.d_blk), _ptr(mt["pk_base"]), _ptr(mt["pk_size"]),
            _ptr(st.blocks), _ptr(mt["packed"]), int(layout), self.sp), "mfb_cg_pack")

    def _multi_wanted(self, n_pts, force=False):
        """True when the blocks exceed shared memory and enough points fill
        the GPU for a multi-point kernel (or it is forced)."""
        st, plan = self.st, self.plan
        nd = plan.ndof.astype(np.int64)
        nl, n_rows = int(plan.n_lambda), int(plan.dof_ptr[-1])
        if int(st.d_cg_local.shape[0]) > 64 or plan.n_sub >= 4095:
            return False
        if force:
            return True
        staged = 8 * (int(np.sum(nd * nd)) + 6 * nl + 2 * n_rows) <= 200 * 1024
        return not staged and n_pts >= 4 * N_SMS

    def _multi_tables(self, n_pts, force=False):
        """Work tables of the 8-points-per-CTA CG (mfb_cg_multi), or None when
        its shared-memory vectors do not fit or the kernel is not wanted."""
        plan, torch = self.plan, self.torch
        nl, n_rows = int(plan.n_lambda), int(plan.dof_ptr[-1])
        if (self.L.mfb_cg_multi_smem(nl, n_rows + 8, 0) + 8192 > 227 * 1024
                or not self._multi_wanted(n_pts, force)):
            return None
        mt = self._pack_tables()
        if "scratch" not in mt:
            mt["n_cta"] = N_SMS
            n = int(self.L.mfb_cg_multi_scratch_doubles(nl, N_SMS))
            mt["scratch"] = torch.empty(n, dtype=torch.float64, device="cuda")
        return mt

    def _cluster_tables(self, n_pts, force=False, shape=None):
        """Tables of the cluster CG (mfb_cg_cluster, cgcluster.py) for the
        first (C, NP) of `shape` (default CLUSTER_SHAPES) whose on-chip
        vectors fit, or None."""
        from . import cgcluster
        torch, st, plan = self.torch, self.st, self.plan
        if not self._multi_wanted(n_pts, force):
            return None
        mt = self._pack_tables()
        cache = st.__dict__.setdefault("_cluster", {})
        for C, NP in (shape or CLUSTER_SHAPES):
            if (C, NP) in cache:
                if cache[(C, NP)] is not None:
                    return cache[(C, NP)]
                continue
            h = mt["host"]
            lay = plan.problem.layout
            centers = np.array([[(b.rect[0] + b.rect[2]) / 2, (b.rect[1] + b.rect[3]) / 2]
                                for b in lay.blocks])
            ct = cgcluster.cluster_tables(plan.n_sub, plan.ndof, plan.dof_ptr, plan.dof_map,
                                          plan.n_lambda, plan.region, centers, C, NP,
                                          h["tasks"], h["sides"], h["pk_base"], h["pk_size"])
            ncl, nr = -1, int(st.d_cg_local.shape[0])
            for flags in (3, 1, 0, 7, 5, 4):   # bit 0 / 1: r / x on chip, bit 2: S p in global
                smem = int(self.L.mfb_cg_cluster_smem(NP, ct["n_used_max"], ct["n_own_max"],
                                                      ct["n_cut_max"], ct["n_cm_max"],
                                                      ct["n_unit_max"], ct["n_strip_max"], nr,
                                                      flags))
                if smem > 220 * 1024:
                    continue
                ncl = int(self.L.mfb_cg_cluster_max_clusters(C, NP, ct["n_own_max"], smem))
                if ncl > 0:
                    break
            if ncl <= 0:
                cache[(C, NP)] = None
                continue
            nv = ncl * C * ct["n_own_max"] * NP
            ct.update(n_clusters=ncl, flags=flags, smem=smem,
                      d_hdr=_dev(ct["hdr"].ravel(), torch.int32),
                      d_tab=_dev(ct["tab"], torch.int32),
                      xs=None if flags & 2 else torch.empty(nv, dtype=torch.float64, device="cuda"),
                      rs=None if flags & 1 else torch.empty(nv, dtype=torch.float64, device="cuda"),
                      ss=None if not flags & 4 else torch.empty(nv, dtype=torch.float64, device="cuda"),
                      seg_counter=torch.zeros(1, dtype=torch.int32, device="cuda"))
            cache[(C, NP)] = ct
            return ct
        return None

    # ------------------------------------------------ (3') S1 CG ------------
    def _s1_tables(self):
        """Item tables of Method S1 (cached on the static state). Item of
        (point k, subdomain s) = k * n_sub + s; its system is the S2 system
        (s, k) = s * n_real + k, whose factors stay in the work buffer."""
        st, plan, torch = self.st, self.plan, self.torch
        t = getattr(st, "_s1", None)
        if t is not None:
            return t
        if st.method != "S2" or st.hwaves or not st.keep_factors or not st.keep_fields:
            raise ValueError("method S1 runs on an S2 sweep state with every system on the "
                             "banded path, factors and fields kept")
        n_real, n_sub = st.reals[1] - st.reals[0], plan.n_sub   # points of this state
        i32, i64 = torch.int32, torch.int64
        woff = np.zeros(len(st.systems), dtype=np.int64)
        for w in st.waves:
            woff[w["idx"]] = w["woff"].cpu().numpy()
        kk, ss = np.meshgrid(np.arange(n_real), np.arange(n_sub), indexing="ij")
        item_sys = (ss * n_real + kk).ravel()
        nout = int(st.out_off[-1])
        item_foff = (kk * nout + st.out_off[:-1][ss]).ravel()
        _, sides, _, _ = cg_tasks(n_sub, plan.ndof.astype(np.int64), plan.dof_ptr, plan.dof_map,
                                  plan.n_lambda)
        # size classes: the long systems (Stokes) and the rest get separate
        # apply launches, each with its own shared-memory footprint, so all
        # items of an iteration are resident at once
        size = np.array([int(p.n + p.nb) for p in plan.patterns])[item_sys // n_real]
        cut = size.max() // 2
        classes = []
        for m in (size > cut, size <= cut):
            ids = np.nonzero(m)[0]
            if len(ids):
                classes.append((_dev(ids.astype(np.int32), i32), len(ids), int(size[ids].max())))
        t = {"n_items": len(item_sys), "item_sys": _dev(item_sys.astype(np.int32), i32),
             "classes": classes,
             "item_hoff": _dev(st.sys_hoff[item_sys], i64),
             "item_foff": _dev(item_foff.astype(np.int64), i64),
             "sides": _dev(np.ascontiguousarray(sides, dtype=np.int32).ravel(), i32),
             "woff": _dev(woff, i64), "fboff": _dev(st.sys_fboff, i64), "nout": nout,
             "max_n": max(int(p.n + p.nb) for p in plan.patterns)}
        st._s1 = t
        return t

    def solve_s1(self, tol, max_iter, hist_cap=None, keep_g=False, check_every=16):
        """Method S1's CG for every point at once (cg_solve with direct_apply,
        interface.py:107-139, 180-194): each iteration is one batched star
        solve of every live (point, subdomain) item with the stored factors,
        then one CG update per point. The host checks the count of running
        points once per `check_every` iterations, one check behind (no stall).
        Returns (lam, iters, status, hist, g) like solve_points."""
        torch, plan, st = self.torch, self.plan, self.st
        t = self._s1_tables()
        n_pts, nl, n_sub = st.reals[1] - st.reals[0], plan.n_lambda, plan.n_sub
        n_items, ldv = t["n_items"], int(plan.ndof.max())
        hist_cap = max_iter if hist_cap is None else hist_cap
        f64, i32 = torch.float64, torch.int32
        x = torch.empty((n_pts, nl), dtype=f64, device="cuda")
        r, p = torch.empty_like(x), torch.empty_like(x)
        scal = torch.empty(2 * n_pts, dtype=f64, device="cuda")
        iters = torch.empty(n_pts, dtype=i32, device="cuda")
        status = torch.empty(n_pts, dtype=i32, device="cuda")
        hist = torch.empty((n_pts, max(hist_cap, 1)), dtype=f64, device="cuda")
        V = torch.empty((n_items, ldv), dtype=f64, device="cuda")
        R = torch.empty((n_items, ldv), dtype=f64, device="cuda")
        live = torch.empty(n_items, dtype=i32, device="cuda")
        nrun = torch.empty(1, dtype=i32, device="cuda")
        g = torch.empty((n_pts, nl), dtype=f64, device="cuda") if keep_g else None
        if self.timing:
            e0 = self._ev()
        self.launches += 1
        _lib.check(self.L.mfb_s1_cg_begin(
            nl, n_pts, n_sub, _ptr(t["sides"]), _ptr(st.hbar), _ptr(t["item_hoff"]), _ptr(x),
            _ptr(r), _ptr(p), _ptr(scal), _ptr(iters), _ptr(status), _ptr(V), ldv, _ptr(live),
            _ptr(nrun), _ptr(g) if keep_g else None, self.sp), "mfb_s1_cg_begin")
        host = torch.empty(2, dtype=i32, pin_memory=True)
        evs = [None, None]
        it, c = 0, 0
        while it < max_iter:
            for _ in range(min(check_every, max_iter - it)):
                self._s1_apply(t, V, ldv, None, 0, R, live)
                _lib.check(self.L.mfb_s1_cg_step(
                    nl, n_pts, n_sub, _ptr(t["sides"]), _ptr(R), ldv, float(tol), int(max_iter),
                    _ptr(x), _ptr(r), _ptr(p), _ptr(scal), _ptr(iters), _ptr(status),
                    _ptr(hist), max(hist_cap, 1), _ptr(V), ldv, _ptr(live), _ptr(nrun), self.sp),
                    "mfb_s1_cg_step")
                self.launches += 1
                it += 1
            slot = c & 1
            with torch.cuda.stream(self.stream):
                host[slot:slot + 1].copy_(nrun, non_blocking=True)
            evs[slot] = torch.cuda.Event()
            evs[slot].record(self.stream)
            prev = evs[slot ^ 1]
            if prev is not None:
                prev.synchronize()
                if int(host[slot ^ 1]) == 0:
                    break
            c += 1
        if self.timing:
            self.cg_events.append((e0, self._ev(), n_pts))
        self._s1_V = V                # every item's lambda restriction (recovery input)
        self._s1_lam = x
        return x, iters, status, hist, g

    def _s1_apply(self, t, V, ldv, X, ldx, R, live):
        """One batched star solve of every item: the long size class on the
        side stream, concurrently with the short one on the engine's."""
        torch, plan, st = self.torch, self.plan, self.st
        cls = t["classes"]
        side = st.side_stream() if len(cls) > 1 else None
        if side is not None:
            side.wait_stream(self.stream)
        for j, (ids, n, max_n) in enumerate(cls):
            sp = ctypes.c_void_p(side.cuda_stream) if (side is not None and j == 0) else self.sp
            self.launches += 1
            _lib.check(self.L.mfb_systems_apply(
                _ptr(plan.pat_dev), n, _ptr(t["item_sys"]), _ptr(st.d_pat), _ptr(st.work),
                _ptr(t["woff"]), _ptr(V), ldv, _ptr(X) if X is not None else None, ldx,
                _ptr(R) if R is not None else None, ldv, max_n,
                _ptr(live) if live is not None else None, _ptr(ids), sp), "mfb_systems_apply")
        if side is not None:
            self.stream.wait_stream(side)

    def s1_fields(self, F):
        """S1's recovery (recover_fields, interface.py:250-260) for this
        state's points: one more batched star solve per (point, subdomain)
        with the final lambda, then the fields bar + star into the rows of
        F (points x every field of every subdomain, rows in point order)."""
        torch, plan, st = self.torch, self.plan, self.st
        t = self._s1_tables()
        ldv, max_n, n_items = int(plan.ndof.max()), t["max_n"], t["n_items"]
        X = torch.empty((n_items, max_n), dtype=torch.float64, device="cuda")
        self._s1_apply(t, self._s1_V, ldv, X, max_n, None, None)
        self.launches += 1
        _lib.check(self.L.mfb_s1_fields(
            _ptr(plan.pat_dev), n_items, _ptr(t["item_sys"]), _ptr(st.d_pat), _ptr(X), max_n,
            _ptr(st.Fb), _ptr(t["fboff"]), _ptr(F), _ptr(t["item_foff"]), self.sp),
            "mfb_s1_fields")

    def s1_moments(self, lam, F):
        """Moments of lambda and of every field over all realizations, in
        realization order (MomentAccumulator, moments.py:25-58), queued like
        moments_launch; finish with moments_finish."""
        torch, plan, st = self.torch, self.plan, self.st
        n_real, nl, nout = plan.grid.n_real, plan.n_lambda, int(st.out_off[-1])
        f64 = torch.float64
        res = torch.empty(3 * nl + 3 * nout, dtype=f64, device="cuda")
        rp = res.data_ptr()
        self.launches += 2
        for n, src, off in ((nl, lam, 0), (nout, F, 3 * nl)):
            _lib.check(self.L.mfb_lambda_moments(
                n, n_real, _ptr(src), _ptr(plan.d_weights), ctypes.c_void_p(rp + 8 * off),
                ctypes.c_void_p(rp + 8 * (off + n)), ctypes.c_void_p(rp + 8 * (off + 2 * n)),
                self.sp), "mfb_lambda_moments")
        keep = 3 * nl + 2 * nout               # the fields' sum of squares stays behind
        host = torch.empty(keep, dtype=f64, pin_memory=True)
        with torch.cuda.stream(self.stream):
            host.copy_(res[:keep], non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.stream)
        tab = st.moment_table(list(range(plan.n_sub)))
        return {"host": host, "res": res, "F": F, "done": done, "tab": tab, "nl": nl,
                "nlm": 3 * nl, "nout": nout, "ng": tab["n"], "with_lambda": True}

    def s1_moments_launch(self):
        """Recovery and moments of a single-state S1 sweep (every point)."""
        torch, plan = self.torch, self.plan
        n_real, nout = plan.grid.n_real, int(self.st.out_off[-1])
        _s1_check_fields(n_real, nout)
        F = torch.empty((n_real, nout), dtype=torch.float64, device="cuda")
        self.s1_fields(F)
        return self.s1_moments(self._s1_lam, F)

    # ----------------------------------------------------- (4) moments ----
    def moments(self, lam, sids=None, with_lambda=True):
        """Moment dict over the "lambda" key (if with_lambda) and the field keys
        of `sids` (default: every subdomain). `lam` holds every point."""
        return self.moments_finish(self.moments_launch(lam, sids, with_lambda))

    def moments_launch(self, lam, sids=None, with_lambda=True):
        """Queue the moment kernels and the device->host copy of their
        results; moments_finish() waits and builds the dict."""
        _check_owner(self.st, "M", "Fb")
        torch, plan, st = self.torch, self.plan, self.st
        nl, n_real = plan.n_lambda, plan.grid.n_real
        f64 = torch.float64
        sids = list(range(plan.n_sub)) if sids is None else list(sids)
        tab = st.moment_table(sids)
        ng = tab["n"]
        # every kernel is launched before the single device->host copy, so
        # the launches queue behind the CG instead of idling the GPU between
        # syncs; the results come back in one pinned transfer
        out_off = tab["out_off"]
        nout = int(out_off[-1]) if ng else 0
        nlm = 3 * nl if with_lambda else 0
        res = torch.empty(nlm + 2 * nout, dtype=f64, device="cuda")
        rp = res.data_ptr()
        if with_lambda:
            self.launches += 1
            _lib.check(self.L.mfb_lambda_moments(
                nl, n_real, _ptr(lam), _ptr(plan.d_weights), ctypes.c_void_p(rp),
                ctypes.c_void_p(rp + 8 * nl), ctypes.c_void_p(rp + 16 * nl),
                self.sp), "mfb_lambda_moments")
        if ng:
            if int(plan.ndof.max()) > MOMENTS_MAX_NDOF:
                raise NativeLibraryError(
                    f"moment kernels hold a subdomain's mortar block in shared memory: "
                    f"{int(plan.ndof.max())} mortar dofs on one subdomain exceed "
                    f"{MOMENTS_MAX_NDOF}")
            W = torch.empty(ng, dtype=f64, device="cuda")
            lstar = torch.empty(st.nv, dtype=f64, device="cuda")
            s_ = torch.empty_like(lstar)
            C = torch.empty(st.nc, dtype=f64, device="cuda")
            self.launches += 3
            _lib.check(self.L.mfb_group_stats(
                ng, _ptr(tab["pat"]), _ptr(tab["gptr"]), _ptr(tab["mem"]), _ptr(plan.d_ndof),
                _ptr(plan.d_dof_ptr), _ptr(plan.d_dof_map), nl, _ptr(lam), _ptr(plan.d_weights),
                _ptr(tab["voff"]), _ptr(tab["coff"]), _ptr(W), _ptr(lstar), _ptr(s_), _ptr(C),
                self.sp), "mfb_group_stats")
            nfb = int(st.Fb.numel())
            fstar = torch.empty(3 * nfb, dtype=f64, device="cuda")
            fp = fstar.data_ptr()
            _lib.check(self.L.mfb_group_fields(
                ng, _ptr(tab["pat"]), _ptr(plan.d_ndof), _ptr(plan.d_nfield), _ptr(st.M),
                _ptr(tab["moff"]), _ptr(st.Fb), _ptr(tab["fboff"]), _ptr(tab["voff"]),
                _ptr(tab["coff"]), _ptr(lstar), _ptr(s_), _ptr(C), ctypes.c_void_p(fp),
                ctypes.c_void_p(fp + 8 * nfb), ctypes.c_void_p(fp + 16 * nfb), self.sp),
                "mfb_group_fields")
            mp = rp + 8 * nlm
            _lib.check(self.L.mfb_moments_reduce(
                len(sids), _ptr(tab["sgptr"]), _ptr(tab["nfield"]), _ptr(tab["fboff"]), _ptr(W),
                ctypes.c_void_p(fp), ctypes.c_void_p(fp + 8 * nfb), ctypes.c_void_p(fp + 16 * nfb),
                st.wtot, _ptr(tab["d_outoff"]), ctypes.c_void_p(mp),
                ctypes.c_void_p(mp + 8 * nout), self.sp), "mfb_moments_reduce")
        host = torch.empty(res.numel(), dtype=f64, pin_memory=True)
        with torch.cuda.stream(self.stream):
            host.copy_(res, non_blocking=True)
        done = torch.cuda.Event()
        done.record(self.stream)
        return {"host": host, "res": res, "done": done, "tab": tab, "nl": nl, "nlm": nlm,
                "nout": nout, "ng": ng, "with_lambda": with_lambda}

    def moments_finish(self, h):
        h["done"].synchronize()
        allh = h["host"].numpy()
        nl, nlm, nout, ng, tab = h["nl"], h["nlm"], h["nout"], h["ng"], h["tab"]
        out = {}
        with_lambda = h["with_lambda"]
        if with_lambda:
            lm = allh[:nlm]
            out["lambda"] = _finalize("lambda", lm[:nl], lm[nl:2 * nl], lm[2 * nl:])
        if not ng:
            return out
        mvh = allh[nlm:]
        mf, vf = mvh[:nout], mvh[nout:].copy()
        # moments.py:43-58 for every key at once: per-key scale, warn, clamp.
        # The scale is >= 1, so nothing can warn unless some entry is below
        # -1e-12: only then are the per-key scales formed.
        keys, starts = tab["keys"], tab["key_start"]
        if len(starts) and vf.min(initial=0.0) < -1e-12:
            sumsq = np.abs(vf + mf * mf)
            scale = np.maximum(1.0, np.maximum.reduceat(sumsq, starts))
            sizes = np.diff(np.append(starts, nout))
            bad = vf < -1e-12 * np.repeat(scale, sizes)
            if bad.any():
                nbad = np.add.reduceat(bad.astype(np.int64), starts)
                for j in np.nonzero(nbad)[0]:
                    seg = vf[starts[j]: starts[j] + sizes[j]]
                    log.warning("field %s: %d variance entries below -1e-12*scale (min %.3e), "
                                "clamping", keys[j], int(nbad[j]), float(seg.min()))
        np.maximum(vf, 0.0, out=vf)
        out.update({key: (mf[a:b].reshape(sh), vf[a:b].reshape(sh))
                    for key, a, b, sh in tab["key_slices"]})
        return out


def _s1_check_fields(n_real, nout):
    need = 8 * n_real * nout
    if need > S1_FIELD_BYTES_MAX:
        raise SizeCapError(f"method S1 keeps every realization's fields on the device: "
                           f"{need / 2 ** 30:.3g} GiB exceeds {S1_FIELD_BYTES_MAX / 2 ** 30:.3g} GiB")


def _finalize(key, mean, var, sumsq):
    """Clamp tiny negative variances like moments.py:43-58."""
    scale = max(1.0, float(np.max(np.abs(sumsq), initial=0.0)))
    bad = var < -1e-12 * scale
    if np.any(bad):
        log.warning("field %s: %d variance entries below -1e-12*scale (min %.3e), "
                    "clamping", key, int(np.sum(bad)), float(var.min()))
    return mean.copy(), np.maximum(var, 0.0)


def run_method(problem, grid, method="S1", tol=1e-9, max_iter=None, workers=1,
               basis_cap_mb=1024.0):
    """Sweep the collocation grid (reference interface.py:288-346), on the device.

    `workers` is accepted for signature compatibility; results do not depend
    on it (the device path is deterministic).
    """
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}, expected one of {METHODS}")
    _lib.lib()                      # raises NativeLibraryError: no CPU fallback
    import torch
    t0 = time.perf_counter()
    n_sub = problem.layout.n_subdomains
    stats = SolveStats.new(method, n_sub)
    stats.n_real = grid.n_real
    nl = problem.space.n_dof
    if max_iter is None:
        max_iter = max(50, 10 * nl)
    plan = get_plan(problem, grid)
    if method != "S1":              # S1 stores no basis (interface.py:313-330)
        _check_basis_cap(plan.basis_bytes(method), basis_cap_mb)
    timings = {"plan": time.perf_counter() - t0}
    if method == "S1":
        # S1 assembles and factors every subdomain per realization like S2
        # (interface.py:316), every system on the banded LU whose factors
        # the star solves reuse: all of them stay resident
        per_real = 8 * sum(int(p.work_doubles + p.x_doubles) for p in plan.patterns)
        cached = plan.__dict__.get("_statics", {}).get(("S2", True))
        if cached is None or cached.darcy_kernel != "band":
            chunk = S1_CHUNK_REALIZATIONS
            if chunk is None:
                free = torch.cuda.mem_get_info()[0]
                chunk = int(0.8 * free // max(per_real, 1))
            if chunk < grid.n_real:
                # too many factors for the device at once: realization chunks
                return _run_s1_chunked(problem, grid, plan, tol, max_iter, stats, timings, t0,
                                       max(chunk, 1))
        eng = SweepEngine(plan, method="S2", darcy_kernel="band", keep_factors=True)
    else:
        eng = SweepEngine(plan, method=method)
    timings["h2d_bytes"] = eng.st.refresh_inputs()
    eng.wave_timing = True          # per-subdomain device time for SolveStats.wall_seconds
    # everything is queued on the stream first (no host round trips between
    # the phases); the verdicts are checked in the reference's order after:
    # singular operators (assembly) before CG failures, moments only then
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(eng.stream)
    eng.kl_fields()
    eng.build_bases()
    ev[1].record(eng.stream)
    if method == "S1":
        lam, iters, status, hist, _ = eng.solve_s1(tol, max_iter)
    else:
        lam, iters, status, hist, _ = eng.solve_points(tol, max_iter)
    ev[2].record(eng.stream)
    cap_error = None
    try:
        mh = eng.s1_moments_launch() if method == "S1" else eng.moments_launch(lam)
    except SizeCapError as e:       # (S1's field cap) raised below, AFTER the verdicts: the
        cap_error, mh = e, None     # reference has no such cap and reports a CG failure first
    ev[3].record(eng.stream)
    # every result travels back in pinned buffers queued behind the moments:
    # one wait, then host-side assembly only
    seg_hist = isinstance(hist, SegmentedHist)
    small_hist = (not seg_hist) and hist.numel() * 8 <= (256 << 20)
    with torch.cuda.stream(eng.stream):
        h_st = torch.empty(status.shape, dtype=status.dtype, pin_memory=True)
        h_it = torch.empty(iters.shape, dtype=iters.dtype, pin_memory=True)
        h_lam = torch.empty(lam.shape, dtype=lam.dtype, pin_memory=True)
        h_st.copy_(status, non_blocking=True)
        h_it.copy_(iters, non_blocking=True)
        h_lam.copy_(lam, non_blocking=True)
        if small_hist:
            h_hist = torch.empty(hist.shape, dtype=hist.dtype, pin_memory=True)
            h_hist.copy_(hist, non_blocking=True)
        if seg_hist:
            h_cnt = torch.empty(1, dtype=torch.int32, pin_memory=True)
            h_cnt.copy_(hist.counter, non_blocking=True)
    eng.check_info()                # syncs the stream: the copies above are done
    st = h_st.numpy()
    it = h_it.numpy()
    if seg_hist and int(h_cnt[0]) > hist.cap:
        # the history pool overflowed (results are complete): rerun the
        # deterministic CG once with the exact pool for the histories
        _, _, _, hist, _ = eng.solve_points(tol, max_iter, hist_segments=int(h_cnt[0]))
    fail = np.nonzero((st == 1) | (st == 2))[0]
    if len(fail):
        k = int(fail[0])
        if seg_hist:
            res = hist.row(k, int(it[k]))
        else:
            res = (h_hist[k] if small_hist else hist[k].cpu()).numpy()[
                :min(int(it[k]), hist.shape[1])].tolist()
        if st[k] == 1:
            raise ConvergenceError(f"interface operator is not positive definite "
                                   f"(p.Sp <= 0 at iteration {int(it[k])}, point {k})",
                                   res[:int(it[k]) - 1])
        raise ConvergenceError(f"CG did not reach tol {tol:g} in {max_iter} iterations "
                               f"(last residual {res[-1]:.3e}, point {k})", res)
    if cap_error is not None:
        raise cap_error
    moments = eng.moments_finish(mh)
    timings["bases"] = ev[0].elapsed_time(ev[1]) / 1e3
    timings["cg"] = ev[1].elapsed_time(ev[2]) / 1e3
    timings["moments"] = ev[2].elapsed_time(ev[3]) / 1e3
    timings["device"] = ev[0].elapsed_time(ev[3]) / 1e3
    timings["launches"] = eng.launches
    lam_h = h_lam.numpy()
    lambdas = list(lam_h)
    if seg_hist:
        residuals = hist.to_host(it.astype(np.int64))
    elif small_hist:
        it_c = np.minimum(it.astype(np.int64), hist.shape[1])
        residuals = ResidualHistories.from_padded(h_hist.numpy(), it_c)
    else:
        residuals = _pack_histories(hist, iters)
    stats.cg_iters = [int(x) for x in it]
    if method == "S1":
        # per realization and subdomain: one factorization, the bar solve,
        # one star solve per CG iteration and the recovery (interface.py:14-16)
        stats.factorizations[:] = grid.n_real
        stats.backsolves[:] = int(np.sum(it.astype(np.int64))) + 2 * grid.n_real
    for s in range(n_sub if method != "S1" else 0):
        # S3: one factorization per (sid, loc); S2: per (sid, realization)
        nloc = int(eng.st.n_loc[s])
        stats.factorizations[s] = nloc
        stats.basis_backsolves[s] = int(plan.ndof[s]) * nloc
        stats.backsolves[s] = int(plan.ndof[s]) * nloc + 2 * grid.n_real
    # per-subdomain time like the reference's (interface.py:142-154: assembly,
    # bases, bar solves, recovery -- not the CG's vector work): the measured
    # device time of the subdomain's basis systems plus an equal share of the
    # moment kernels (the recovery of every subdomain's fields)
    stats.wall_seconds[:] = eng.subdomain_seconds(n_sub) + timings["moments"] / max(n_sub, 1)
    timings["total"] = time.perf_counter() - t0
    return RunResult(moments, stats, lambdas, residuals, grid, timings)


def _run_s1_chunked(problem, grid, plan, tol, max_iter, stats, timings, t0, chunk):
    """Method S1 in realization chunks when the factors of every (subdomain,
    realization) do not fit on the device at once: each chunk assembles and
    factors its realizations (an S2 state restricted to them), runs their
    CG and recovery, and writes its rows of lambda and of the fields; the
    moments run once over all rows in realization order, so the result does
    not depend on the chunking. Verdicts in the reference's order: the first
    chunk holding a singular operator or a failed point raises."""
    import torch
    n_real, nl = grid.n_real, plan.n_lambda
    nout = int(np.sum(plan.nfield.astype(np.int64)))
    _s1_check_fields(n_real, nout)
    f64 = torch.float64
    lam_all = torch.empty((n_real, nl), dtype=f64, device="cuda")
    F = torch.empty((n_real, nout), dtype=f64, device="cuda")
    it_all = np.zeros(n_real, dtype=np.int64)
    hists = []
    timings["chunks"] = 0
    eng = None
    for r0 in range(0, n_real, chunk):
        r1 = min(n_real, r0 + chunk)
        eng = None                              # the previous chunk's factors go first
        torch.cuda.empty_cache()
        eng = SweepEngine(plan, method="S2", darcy_kernel="band", keep_factors=True,
                          reals=(r0, r1))
        eng.kl_fields()
        eng.build_bases()
        lam, iters, status, hist, _ = eng.solve_s1(tol, max_iter)
        eng.check_info()                        # syncs: singular operators first
        st_h, it_h = status.cpu().numpy(), iters.cpu().numpy()
        fail = np.nonzero((st_h == 1) | (st_h == 2))[0]
        if len(fail):
            j = int(fail[0])
            res = hist[j].cpu().numpy()[:min(int(it_h[j]), hist.shape[1])].tolist()
            k = r0 + j
            if st_h[j] == 1:
                raise ConvergenceError(f"interface operator is not positive definite "
                                       f"(p.Sp <= 0 at iteration {int(it_h[j])}, point {k})",
                                       res[:int(it_h[j]) - 1])
            raise ConvergenceError(f"CG did not reach tol {tol:g} in {max_iter} iterations "
                                   f"(last residual {res[-1]:.3e}, point {k})", res)
        lam_all[r0:r1].copy_(lam)
        eng.s1_fields(F[r0:r1])
        it_all[r0:r1] = it_h
        hists.append(_pack_histories(hist, iters))
        timings["chunks"] += 1
    mh = eng.s1_moments(lam_all, F)
    moments = eng.moments_finish(mh)
    flat = np.concatenate([h.array(j) for h in hists for j in range(len(h))]) \
        if n_real else np.zeros(0)
    residuals = ResidualHistories(flat, np.minimum(it_all, max_iter))
    stats.cg_iters = [int(x) for x in it_all]
    stats.factorizations[:] = n_real
    stats.backsolves[:] = int(it_all.sum()) + 2 * n_real
    stats.wall_seconds[:] = (time.perf_counter() - t0) / max(plan.n_sub, 1)
    timings["total"] = time.perf_counter() - t0
    return RunResult(moments, stats, list(lam_all.cpu().numpy()), residuals, grid, timings)
