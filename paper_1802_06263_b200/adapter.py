"""Read-only views of the reference's host objects that the device tables need.

The drop-in takes the caller's own `sdmortar` objects -- `StokesDarcyProblem`
(problem.py:25-38: layout, meshes, space, perm, physics, bcs, sources, and
the derived traces / couplings / kl_cells of its __post_init__) and
`CollocationGrid` (collocation.py:44-72) -- and never rebuilds them. The
helpers below derive, from those objects' public attributes only, the few
quantities the table builders (discretization.py, hybrid.py, plan.py) need in
array form. Each one restates the reference expression it mirrors, so the
device tables carry the same bits the reference's assembly would compute.
"""

import numpy as np

from ._ref import sdmortar

_darcy, _geometry, _stokes = sdmortar.darcy, sdmortar.geometry, sdmortar.stokes

SIDES = _darcy.SIDES                          # darcy.py:25
OUTWARD_SIGN = _geometry.OUTWARD_SIGN         # geometry.py:268-269
P2_EDGE_MASS = _stokes.EDGE_MASS                # stokes.py:38 (P2 edge mass / L)
DarcyBC = _darcy.DarcyBC                      # darcy.py:28-34
StokesBC = _stokes.StokesBC                   # stokes.py:66-71


def darcy_sids(problem):
    """Darcy subdomain ids in ascending order (problem.permeability's loop,
    problem.py:85-96)."""
    lay = problem.layout
    return [s for s in range(lay.n_subdomains) if lay.physics(s) == "darcy"]


def mode_table(perm, region, x, y):
    """(Phi, mean) of one KL region at points: Phi[c, j] = sqrt(lam_j) f_j(x_c)
    (KLRegionExpansion.evaluate_modes, random_field.py:125-140) and the mean
    log-permeability (MeanLogPerm.__call__, 200-209) -- the realization-
    independent inputs of LogPermField.evaluate_log (232-238)."""
    exp = perm.regions[region]
    phi = exp.evaluate_modes(x, y) if exp.n_term else np.zeros((len(x), 0))
    return phi, perm.mean(x, y, region=region)


def cell_edge_table(mesh):
    """(n_cells, 4) edge ids (west, east, south, north) in cell order:
    DarcyMesh.cell_edges (geometry.py:238-245) for every cell(ix, iy) =
    iy*nx + ix, vectorised."""
    iy, ix = np.divmod(np.arange(mesh.n_cells), mesh.nx)
    v = iy * (mesh.nx + 1) + ix
    h = mesh.n_vedges + iy * mesh.nx + ix
    return np.stack([v, v + 1, h, h + mesh.nx], axis=1)


def edge_midpoint(mesh, e):
    """Midpoint of Darcy edge e, the point the pressure data g is sampled at
    (DarcyOperator._edge_mid, darcy.py:209-217; same arithmetic)."""
    x0, y0 = mesh.rect[0], mesh.rect[1]
    if e < mesh.n_vedges:
        iy, ix = divmod(int(e), mesh.nx + 1)
        return (x0 + ix * mesh.hx, y0 + (iy + 0.5) * mesh.hy)
    iy, ix = divmod(int(e) - mesh.n_vedges, mesh.nx)
    return (x0 + (ix + 0.5) * mesh.hx, y0 + iy * mesh.hy)


def load_config(path):
    """(problem, grid, options) of a JSON config file, built by the reference
    itself: sdmortar.config.parse_config + build_from_config with the file's
    directory (the same two calls as sdmortar.driver.run_file, driver.py:32-36)."""
    import os
    from sdmortar.config import build_from_config, parse_config
    return build_from_config(parse_config(path), os.path.dirname(os.path.abspath(path)))
