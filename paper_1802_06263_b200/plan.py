"""Device plan: the problem's realization-independent data resident in HBM.

`DevicePlan(problem, grid)` flattens the host setup into device tensors once
per (problem, grid): per-subdomain system patterns (discretization.py), the
KL mode tables, mortar dof maps, local-index tables and the S3 group member
lists. PyTorch is used only as the allocator/stream provider; all compute
goes through the sm_100a library (`_lib.py`).
"""

import ctypes

import os

import numpy as np

from . import _lib
from .discretization import darcy_pattern, stokes_pattern
from .hybrid import assembly_tables, hybrid_pattern
from .adapter import darcy_sids, mode_table


def _dev(a, dtype):
    import torch
    t = torch.as_tensor(np.ascontiguousarray(a), dtype=dtype)
    return t.to("cuda", non_blocking=False)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None and t.numel() else ctypes.c_void_p(0)


def _host_map(fn, items):
    """fn over items on up to 8 host threads, results in order."""
    items = list(items)
    workers = min(8, len(os.sched_getaffinity(0)), len(items))
    if workers <= 1:
        return [fn(i) for i in items]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(fn, items))


class HostTables:
    """The realization-independent host tables of (problem, grid), before upload.

    Built from the reference's own objects (`sdmortar` StokesDarcyProblem and
    CollocationGrid: layout, meshes, space, perm, couplings, traces, bcs,
    kl_cells, local tables) through `adapter.py`; `DevicePlan` uploads them.
    `arrays()` flattens every table into name -> ndarray (tests hash them).
    """

    def __init__(self, problem, grid):
        lay = problem.layout
        self.n_sub = lay.n_subdomains
        self.n_lambda = problem.space.n_dof
        self.darcy = darcy_sids(problem)
        # concatenated mean-field K layout over Darcy subdomains
        self.k0_off, off = {}, 0
        for s in self.darcy:
            self.k0_off[s] = off
            off += problem.meshes[s].n_cells
        self.k0_len = off
        # host K0 (exp(mean)) only for the Stokes kernel-structure test
        K0_host = np.zeros(self.k0_len)
        for s in self.darcy:
            c = problem.meshes[s].centroids
            _, mean = mode_table(problem.perm, lay.blocks[s].kl_region, c[:, 0], c[:, 1])
            K0_host[self.k0_off[s]:self.k0_off[s] + len(mean)] = np.exp(mean)
        # per-subdomain tables are independent: built on a few host threads
        # (the sorts and concatenations inside release the GIL), same tables
        def pattern(sid):
            if lay.physics(sid) == "darcy":
                return darcy_pattern(problem, sid)
            return stokes_pattern(problem, sid, self.k0_off, K0_host)
        self.patterns = _host_map(pattern, range(self.n_sub))
        self.ndof = np.array([p.ndof for p in self.patterns], dtype=np.int32)
        self.nfield = np.array([p.nfield for p in self.patterns], dtype=np.int32)
        dofs = [problem.space.sub_dofs(lay, s) for s in range(self.n_sub)]
        self.dof_ptr = np.cumsum([0] + [len(d) for d in dofs]).astype(np.int32)
        self.dof_map = np.concatenate(dofs).astype(np.int32)
        self.region = np.array([lay.blocks[s].kl_region if lay.physics(s) == "darcy" else -1
                                for s in range(self.n_sub)], dtype=np.int32)
        self.n_loc = np.array([grid.local_counts[r] if r >= 0 else 1 for r in self.region],
                              dtype=np.int64)
        self.hyb = dict(zip(self.darcy, _host_map(lambda s: hybrid_pattern(problem, s),
                                                  self.darcy)))
        self.hyb_panel = {s: h.choose_panel() for s, h in self.hyb.items()}
        self.kl_modes = {}
        for s in self.darcy:
            c = problem.meshes[s].centroids
            self.kl_modes[s] = mode_table(problem.perm, lay.blocks[s].kl_region,
                                          c[:, 0], c[:, 1])
        self.local = (np.stack(grid.local_indices).astype(np.int32) if grid.local_indices
                      else np.zeros((1, grid.n_real), dtype=np.int32))
        self.weights = np.ascontiguousarray(grid.weights, dtype=np.float64)

    def arrays(self):
        """name -> ndarray of every table (patterns, hybrid patterns and their
        assembly tables, KL mode tables, dof maps, local tables)."""
        out = {"ndof": self.ndof, "nfield": self.nfield, "dof_ptr": self.dof_ptr,
               "dof_map": self.dof_map, "region": self.region, "n_loc": self.n_loc,
               "local": self.local, "weights": self.weights}

        def add(prefix, obj):
            for k, v in sorted(vars(obj).items()):
                if isinstance(v, np.ndarray):
                    out[f"{prefix}.{k}"] = v
                elif isinstance(v, (int, float, np.integer, np.floating)) and \
                        not isinstance(v, bool):
                    out[f"{prefix}.{k}"] = np.array(v)
        for s, p in enumerate(self.patterns):
            add(f"pat{s}", p)
        for s, h in self.hyb.items():
            add(f"hyb{s}", h)
            for k, v in assembly_tables(h).items():
                out[f"hyb{s}.asm.{k}"] = np.asarray(v)
            out[f"hyb{s}.panel"] = np.array(self.hyb_panel[s])
        for s, (phi, mean) in self.kl_modes.items():
            out[f"kl{s}.phi"], out[f"kl{s}.mean"] = phi, mean
        return out


class DevicePlan:
    """Everything about (problem, grid) that does not depend on lambda."""

    def __init__(self, problem, grid):
        import torch
        self.torch = torch
        self.problem, self.grid = problem, grid
        ht = HostTables(problem, grid)
        self.host = ht
        for name in ("n_sub", "n_lambda", "darcy", "k0_off", "k0_len", "patterns", "ndof",
                     "nfield", "dof_ptr", "dof_map", "region", "n_loc", "hyb", "hyb_panel"):
            setattr(self, name, getattr(ht, name))
        self._upload_patterns()
        self._upload_hybrid()
        self._upload_tables()

    # ---------------------------------------------------------------- upload
    def _upload_patterns(self):
        torch = self.torch
        i32, f64, i64 = torch.int32, torch.float64, torch.int64
        self._keep = []
        structs = (_lib.MfbPattern * self.n_sub)()
        for s, p in enumerate(self.patterns):
            arrs = {
                "e_row": _dev(p.e_row, i32), "e_col": _dev(p.e_col, i32),
                "e_tptr": _dev(p.e_tptr, i32), "t_kind": _dev(p.t_kind, i32),
                "t_c": _dev(p.t_c, f64), "t_k": _dev(p.t_k, i32),
                "E": _dev(p.E.ravel(), f64), "G": _dev(p.G.ravel(), f64),
                "q_ptr": _dev(p.q_ptr, i32), "q_row": _dev(p.q_row, i32),
                "q_val": _dev(p.q_val, f64), "bar_const": _dev(p.bar_const, f64),
                "b_row": _dev(p.b_row, i32), "b_tptr": _dev(p.b_tptr, i32),
                "bt_kind": _dev(p.bt_kind, i32), "bt_c": _dev(p.bt_c, f64),
                "bt_k": _dev(p.bt_k, i32), "h_lift": _dev(p.h_lift, f64),
                "p_ptr": _dev(p.p_ptr, i32), "p_col": _dev(p.p_col, i32),
                "p_val": _dev(p.p_val, f64), "f_lift": _dev(p.f_lift, f64),
            }
            self._keep.append(arrs)
            st = structs[s]
            st.n, st.kl, st.ku, st.ldab = p.n, p.kl, p.ku, p.ldab
            st.nb, st.ndof, st.nfield = p.nb, p.ndof, p.nfield
            st.n_entries = len(p.e_row)
            st.n_bar_rows = len(p.b_row)
            for name, t in arrs.items():
                setattr(st, name, _ptr(t).value or 0)
        raw = bytes(structs)
        host = torch.frombuffer(bytearray(raw), dtype=torch.uint8)
        self.pat_dev = host.to("cuda")

    def _upload_hybrid(self):
        """MfbHybPattern per subdomain (Darcy entries filled; index = sid)."""
        torch = self.torch
        i32, f64 = torch.int32, torch.float64
        structs = (_lib.MfbHybPattern * self.n_sub)()
        self._keep_h = []
        for s, h in self.hyb.items():
            # transpose of G: mortar dof -> (interface edge id, coefficient)
            gam_edge = np.nonzero(h.edge_kind == 1)[0]
            order = np.argsort(h.edge_idx[gam_edge])
            gam_edge = gam_edge[order]
            rows = np.repeat(gam_edge, np.diff(h.gam_ptr))
            o = np.argsort(h.gam_d, kind="stable")
            dof_ptr = np.zeros(h.ndof + 1, dtype=np.int64)
            np.add.at(dof_ptr, h.gam_d + 1, 1)
            dof_ptr = np.cumsum(dof_ptr)
            arrs = {
                "row_edge": _dev(h.row_edge, i32), "edge_kind": _dev(h.edge_kind, i32),
                "edge_idx": _dev(h.edge_idx, i32), "edge_cells": _dev(h.edge_cells.ravel(), i32),
                "edge_slot": _dev(h.edge_slot.ravel(), i32),
                "edge_noflow": _dev(h.edge_noflow, i32),
                "cell_edges": _dev(h.cell_edges.ravel(), i32),
                "gam_ptr": _dev(h.gam_ptr, i32), "gam_d": _dev(h.gam_d, i32),
                "gam_c": _dev(h.gam_c, f64), "dof_ptr": _dev(dof_ptr, i32),
                "dof_edge": _dev(rows[o], i32), "dof_coef": _dev(h.gam_c[o], f64),
                "p_val": _dev(h.p_val, f64), "src_k": _dev(h.src_k.ravel(), f64),
                "src_c": _dev(h.src_c.ravel(), f64), "cell_f": _dev(h.cell_f.ravel(), f64),
                "cell_q": _dev(h.cell_q, f64),
            }
            T = assembly_tables(h)
            asm_row = np.repeat(np.arange(h.n), np.diff(T["asm_ptr"]))
            arrs.update({
                "asm_ptr": _dev(T["asm_ptr"], i32), "asm_row": _dev(asm_row, i32),
                "asm_dest": _dev(T["asm_dest"], i32), "asm_tptr": _dev(T["asm_tptr"], i32),
                "asm_cell": _dev(T["asm_cell"], i32), "asm_coef": _dev(T["asm_coef"], f64),
                "z_dest": _dev(T["z_dest"], i32), "z_tptr": _dev(T["z_tptr"], i32),
                "z_cell": _dev(T["z_cell"], i32), "z_coef": _dev(T["z_coef"], f64)})
            pe_ptr, pe_rec, pe_coef = h.panel_entries(self.hyb_panel[s])
            arrs.update({"pe_ptr": _dev(pe_ptr, i32), "pe_rec": _dev(pe_rec.ravel(), i32),
                         "pe_coef": _dev(pe_coef.ravel(), f64)})
            self._keep_h.append(arrs)
            st = structs[s]
            ws = h.layout_for(self.hyb_panel[s])[0]
            st.n, st.w, st.ws, st.ndof, st.nfield = h.n, h.w, ws, h.ndof, h.nfield
            st.n_edges, st.n_cells = len(h.edge_kind), len(h.cell_q)
            st.has_src = int(h.has_src)
            st.z_n = int(len(T["z_dest"]))
            st.hx, st.hy, st.nu = h.hx, h.hy, h.nu
            st.s2 = h.hx * h.hx + h.hy * h.hy
            for i, v in enumerate(h.Hhat.ravel()):
                st.Hhat[i] = float(v)
            for name, t in arrs.items():
                setattr(st, name, _ptr(t).value or 0)
        raw = bytes(structs)
        self.hyb_dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to("cuda")

    def _upload_tables(self):
        torch = self.torch
        g = self.grid
        self.d_ndof = _dev(self.ndof, torch.int32)
        self.d_nfield = _dev(self.nfield, torch.int32)
        self.d_dof_ptr = _dev(self.dof_ptr, torch.int32)
        self.d_dof_map = _dev(self.dof_map, torch.int32)
        self.d_region = _dev(self.region, torch.int32)
        li = np.stack(g.local_indices).astype(np.int32) if g.local_indices else \
            np.zeros((1, g.n_real), dtype=np.int32)
        self.d_local = _dev(li, torch.int32)
        self.d_weights = _dev(g.weights, torch.float64)

    # ---------------------------------------------------------- system list
    def s3_systems(self):
        """(sid, loc) of every S3 basis system, sid-major (interface.py:357-373)."""
        out = []
        for s in range(self.n_sub):
            out += [(s, l) for l in range(int(self.n_loc[s]))]
        return out

    def sweep_static(self, keep_fields=True, darcy_kernel="hybrid", method="S3",
                     keep_factors=False, reals=None):
        """Resident sweep state for `method` ("S3" or "S2"), cached per method.
        keep_factors: every banded system keeps its own work region (its LU
        stays for later solves, mfb_systems_apply). reals = (r0, r1): an S2
        state for realizations r0..r1-1 only, built fresh and not cached
        (Method S1's realization chunks)."""
        if reals is not None:
            from .interface import _SweepStatic
            return _SweepStatic(self, keep_fields, darcy_kernel, method, keep_factors, reals)
        cache = self.__dict__.setdefault("_statics", {})
        key = (method, keep_factors)
        st = cache.get(key)
        if (st is None or (keep_fields and not st.keep_fields)
                or st.darcy_kernel != darcy_kernel):
            from .interface import _SweepStatic
            cache.pop(key, None)
            st = _SweepStatic(self, keep_fields, darcy_kernel, method, keep_factors)
            cache[key] = st
        return st

    def basis_bytes(self, method="S3"):
        """Basis storage the reference's size cap checks (interface.py:271-276):
        S3 the whole per-(sid, loc) pool (375), S2 one realization (320-322)."""
        if method == "S2":
            return [8 * int(self.ndof[s]) ** 2 for s in range(self.n_sub)]
        return [8 * int(self.ndof[s]) ** 2 * int(self.n_loc[s]) for s in range(self.n_sub)]
