"""ctypes binding of the sm_100a library `_mfb.so` (C ABI in include/mfb.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, `lib()` raises NativeLibraryError.
"""

import ctypes
import os

from .errors import NativeLibraryError

_SO = os.environ.get("MFB_LIBRARY") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_mfb.so")
_lib = None

_p = ctypes.c_void_p
_i = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double


class MfbPattern(ctypes.Structure):
    _fields_ = [
        ("n", _i), ("kl", _i), ("ku", _i), ("ldab", _i), ("nb", _i), ("ndof", _i),
        ("nfield", _i), ("n_entries", _i),
        ("e_row", _p), ("e_col", _p), ("e_tptr", _p), ("t_kind", _p), ("t_c", _p),
        ("t_k", _p), ("E", _p), ("G", _p), ("q_ptr", _p), ("q_row", _p), ("q_val", _p),
        ("bar_const", _p), ("n_bar_rows", _i), ("b_row", _p), ("b_tptr", _p),
        ("bt_kind", _p), ("bt_c", _p), ("bt_k", _p), ("h_lift", _p), ("p_ptr", _p),
        ("p_col", _p), ("p_val", _p), ("f_lift", _p),
    ]


class MfbKlTable(ctypes.Structure):
    _fields_ = [("phi", _p), ("mean", _p), ("xi", _p), ("dst0", _ll), ("dst", _ll), ("ld", _ll),
                ("n_cells", _i), ("n_term", _i), ("n_rows", _i), ("pad", _i)]


class MfbHybPattern(ctypes.Structure):
    _fields_ = [
        ("n", _i), ("w", _i), ("ws", _i), ("ndof", _i), ("nfield", _i), ("n_edges", _i),
        ("n_cells", _i), ("has_src", _i), ("hx", _d), ("hy", _d), ("nu", _d), ("s2", _d),
        ("Hhat", _d * 16),
        ("row_edge", _p), ("edge_kind", _p), ("edge_idx", _p), ("edge_cells", _p),
        ("edge_slot", _p), ("edge_noflow", _p), ("cell_edges", _p), ("gam_ptr", _p),
        ("gam_d", _p), ("gam_c", _p), ("dof_ptr", _p), ("dof_edge", _p), ("dof_coef", _p),
        ("p_val", _p), ("src_k", _p), ("src_c", _p), ("cell_f", _p), ("cell_q", _p),
        ("z_n", _i), ("asm_ptr", _p), ("asm_row", _p), ("asm_dest", _p), ("asm_tptr", _p),
        ("asm_cell", _p), ("asm_coef", _p), ("z_dest", _p), ("z_tptr", _p), ("z_cell", _p),
        ("z_coef", _p), ("pe_ptr", _p), ("pe_rec", _p), ("pe_coef", _p),
    ]


_SIGS = {
    "mfb_version": ([], ctypes.c_char_p),
    "mfb_strerror": ([_i], ctypes.c_char_p),
    "mfb_kl_realize": ([_p, _p, _i, _i, _p, _i, _p, _p], _i),
    "mfb_kl_realize_ld": ([_p, _p, _i, _i, _p, _i, _p, _ll, _p], _i),
    "mfb_kl_realize_batched": ([_i, _p, _i, _i, _p, _p], _i),
    "mfb_systems_solve": ([_p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _i, _p, _i, _p], _i),
    "mfb_systems_extract": ([_p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p], _i),
    "mfb_blocks_symmetrize": ([_p, _i, _p, _p, _p, _p], _i),
    "mfb_cg_batched": ([_i, _i, _p, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i, _i, _d, _i,
                        _p, _p, _p, _p, _i, _p, ctypes.c_longlong, _i, _p], _i),
    "mfb_systems_apply": ([_p, _i, _p, _p, _p, _p, _p, _ll, _p, _ll, _p, _ll, _i, _p, _p, _p],
                          _i),
    "mfb_s1_cg_begin": ([_i, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _ll, _p, _p, _p,
                         _p], _i),
    "mfb_s1_cg_step": ([_i, _i, _i, _p, _p, _ll, _d, _i, _p, _p, _p, _p, _p, _p, _p, _i, _p,
                        _ll, _p, _p, _p], _i),
    "mfb_s1_fields": ([_p, _i, _p, _p, _p, _ll, _p, _p, _p, _p, _p], _i),
    "mfb_cg_multi_scratch_doubles": ([_i, _i], _ll),
    "mfb_cg_multi_smem": ([_i, _i, _i], _ll),
    "mfb_cg_multi": ([_i, _i, _i, _p, _p, _p, _p, _i, _p, _p, _p, _i, _p, _p, _i, _i, _d, _i,
                      _p, _p, _p, _p, _i, _p, _p, _i, _p, _p, _p, _p, _i, _p, _p, _p, _i, _ll,
                      _p, _p, _p, _i, _i, _p, _i, _p], _i),
    "mfb_cg_pack": ([_i, _p, _p, _p, _i, _p, _p, _p, _p, _p, _i, _p], _i),
    "mfb_basis_apply": ([_i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p], _i),
    "mfb_debug_cluster": ([_i], _i),
    "mfb_debug_multi": ([_i, _p], _i),
    "mfb_debug_multi_warps": ([_p, _i], _i),
    "mfb_debug_cluster_prof": ([_p, _i], _i),
    "mfb_cg_cluster_max_clusters": ([_i, _i, _i, _ll], _i),
    "mfb_cg_cluster_smem": ([_i, _i, _i, _i, _i, _i, _i, _i, _i], _ll),
    "mfb_cg_cluster": ([_i, _i, _i, _p, _p, _i, _i, _i, _i, _i, _i, _i, _ll, _p, _p, _i, _p, _p, _i, _p,
                        _p, _p, _i, _i, _d, _i, _p, _p, _p, _p, _p, _p, _p, _i, _p, _p, _i, _ll,
                        _p, _i, _p, _p], _i),
    "mfb_group_stats": ([_i, _p, _p, _p, _p, _p, _p, _i, _p, _p, _p, _p, _p, _p, _p, _p,
                         _p], _i),
    "mfb_group_fields": ([_i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p,
                          _p], _i),
    "mfb_moments_reduce": ([_i, _p, _p, _p, _p, _p, _p, _p, _d, _p, _p, _p, _p], _i),
    "mfb_lambda_moments": ([_i, _i, _p, _p, _p, _p, _p, _p], _i),
    "mfb_selftest_dmma": ([_p, _p], _i),
    "mfb_debug_prof": ([_p], _i),
    "mfb_debug_bprof": ([_p], _i),
    "mfb_debug_timeline": ([_p], _i),
    "mfb_debug_cgprof": ([_p], _i),
    "mfb_darcy_condense": ([_p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _i, _i, _p], _i),
    "mfb_darcy_backsolve": ([_p, _i, _p, _p, _p, _p, _p, _i, _i, _p], _i),
    "mfb_darcy_recover": ([_p, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p], _i),
}


def exported_symbols():
    return sorted(_SIGS)


def load(path=_SO):
    """Open the shared library and declare signatures (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} is missing; build it with `python -m paper_1802_06263_b200._build` "
            f"(there is no CPU fallback)")
    lib_ = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib_, name)
        fn.argtypes = args
        fn.restype = res
    _check_provenance(lib_, path)
    _lib = lib_
    return _lib


def _check_provenance(lib_, path):
    """The library must have been built from the sources in this tree
    (mfb_version carries the source hash _build embedded). A library built
    elsewhere (MFB_LIBRARY, experiments) is accepted only with
    MFB_ALLOW_FOREIGN_LIBRARY=1."""
    from . import _build
    ver = lib_.mfb_version().decode()
    built = ver.rsplit(" src ", 1)[-1] if " src " in ver else "unknown"
    if not _build.source_files():
        return                                  # sources not shipped: nothing to compare
    tree = _build.source_hash()
    if built != tree and os.environ.get("MFB_ALLOW_FOREIGN_LIBRARY") != "1":
        raise NativeLibraryError(
            f"{path} was built from sources {built}, the tree is {tree}: rebuild with "
            f"`python -m paper_1802_06263_b200._build --force`")


def lib():
    """The loaded library, after checking a CUDA device is usable."""
    import torch
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device: the B200 path has no CPU fallback")
    return load()


def check(code, what):
    if code != 0:
        msg = load().mfb_strerror(code).decode()
        raise NativeLibraryError(f"{what} failed: {msg} (code {code})")
