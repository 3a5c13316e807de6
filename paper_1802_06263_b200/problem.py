"""The realization-independent problem: layout, meshes, mortars, traces, data.

Mirrors the reference's `StokesDarcyProblem` (problem.py:25-81) plus the
trace bookkeeping of `darcy.interface_trace` (darcy.py:38-55) and
`stokes.interface_trace` (stokes.py:66-105). Everything here is host setup;
`plan.py` flattens it into the index/coefficient arrays the device consumes.
"""

from dataclasses import dataclass, field

import numpy as np

from .geometry import (OUTWARD_SIGN, build_subdomain_mesh, edges_on_span,
                       side_of_interface)
from .mortar import build_side_coupling


@dataclass(frozen=True)
class Physics:
    nu_s: float = 1.0
    nu_d: float = 1.0
    alpha: float = 1.0


@dataclass(frozen=True)
class DarcyBC:
    kind: str  # "noflow" | "pressure"
    value: object = None  # callable (x, y) or None (-> 0)


@dataclass(frozen=True)
class StokesBC:
    kind: str  # "velocity" | "stress"
    value: object = None  # callable (x, y) -> (vx, vy) or None (-> 0)


@dataclass(frozen=True)
class DarcyTrace:
    """Fine Darcy edges on one interface, in tangent order."""

    iface: int
    edges: np.ndarray
    sigma_out: int  # +1 if the fixed +x/+y edge orientation points outward
    normal_sign: int
    s_breaks: np.ndarray


@dataclass(frozen=True)
class StokesTrace:
    """P2 edge triples and trace nodes of one Stokes side of an interface."""

    iface: int
    kind: str
    edges: list
    nodes: np.ndarray
    s_breaks: np.ndarray
    sigma: int  # +1 on the lower-id side
    normal: tuple
    tangent: tuple


def darcy_trace(mesh, block, iface):
    side = side_of_interface(block, iface)
    brk = mesh.side_breaks(side)
    idx = edges_on_span(brk, iface.span)
    s = brk[idx[0]:idx[-1] + 2] - iface.span[0]
    return DarcyTrace(iface.index, mesh.boundary_edges(side)[idx],
                      OUTWARD_SIGN[side], iface.normal_sign, s)


def stokes_trace(mesh, block, iface, sid):
    side = side_of_interface(block, iface)
    brk = mesh.side_breaks(side)
    idx = edges_on_span(brk, iface.span)
    sides = mesh.boundary_edges(side)
    edges = [sides[k] for k in idx]
    nodes = [edges[0][0]] + [n for e in edges for n in e[1:]]
    s = brk[idx[0]:idx[-1] + 2] - iface.span[0]
    return StokesTrace(iface.index, iface.kind, edges, np.array(nodes), s,
                       iface.side_sign(sid), tuple(iface.normal),
                       tuple(iface.tangent))


@dataclass
class StokesDarcyProblem:
    layout: object
    meshes: dict
    space: object
    perm: object
    physics: Physics
    bcs: dict
    f_s: object = None
    f_d: object = None
    q_d: object = None
    traces: dict = field(init=False)
    couplings: dict = field(init=False)
    kl_cells: dict = field(init=False)

    def __post_init__(self):
        lay = self.layout
        self.traces = {sid: [] for sid in range(lay.n_subdomains)}
        self.couplings = {}
        self.kl_cells = {}
        for g in lay.interfaces:
            for sid in (g.i, g.j):
                blk, mesh = lay.blocks[sid], self.meshes[sid]
                if blk.physics == "darcy":
                    tr, kind = darcy_trace(mesh, blk, g), "darcy"
                else:
                    tr, kind = stokes_trace(mesh, blk, g, sid), "stokes"
                self.traces[sid].append(tr)
                self.couplings[(g.index, sid)] = build_side_coupling(
                    self.space.block(g.index), tr.s_breaks, kind)
            if g.kind == "sd":
                s_sid = g.i if lay.physics(g.i) == "stokes" else g.j
                d_sid = g.j if s_sid == g.i else g.i
                self.kl_cells.setdefault(s_sid, {})[g.index] = (
                    d_sid, self._bjs_cells(s_sid, d_sid, g))

    def trace(self, sid, iface_index):
        return next(t for t in self.traces[sid] if t.iface == iface_index)

    def _bjs_cells(self, s_sid, d_sid, iface):
        """Darcy cell under each fine Stokes edge midpoint (problem.py:65-81)."""
        tr = self.trace(s_sid, iface.index)
        dm = self.meshes[d_sid]
        db = self.layout.blocks[d_sid]
        dside = side_of_interface(db, iface)
        mids = iface.span[0] + 0.5 * (tr.s_breaks[:-1] + tr.s_breaks[1:])
        out = np.empty(len(mids), dtype=int)
        for k, m in enumerate(mids):
            if iface.axis == "y":
                ix = int(np.clip((m - db.x0) / dm.hx, 0, dm.nx - 1))
                iy = dm.ny - 1 if dside == "top" else 0
            else:
                iy = int(np.clip((m - db.y0) / dm.hy, 0, dm.ny - 1))
                ix = dm.nx - 1 if dside == "right" else 0
            out[k] = dm.cell(ix, iy)
        return out

    def darcy_sids(self):
        return [s for s in range(self.layout.n_subdomains)
                if self.layout.physics(s) == "darcy"]

    def cell_centers(self, sid):
        mesh = self.meshes[sid]
        if self.layout.physics(sid) == "darcy":
            return mesh.centroids
        return mesh.tri_vertices.mean(axis=1)


def build_problem(layout, space, perm, physics, bcs, f_s=None, f_d=None,
                  q_d=None, meshes=None):
    if meshes is None:
        meshes = {sid: build_subdomain_mesh(b) for sid, b in enumerate(layout.blocks)}
    return StokesDarcyProblem(layout, meshes, space, perm, physics, bcs,
                              f_s=f_s, f_d=f_d, q_d=q_d)
