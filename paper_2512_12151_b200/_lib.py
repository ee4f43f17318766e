"""ctypes binding of libibf.so (include/ibf.h) — the only way into the kernels.

There is no CPU fallback: importing the compute entry points without the
built library, or calling them without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# IBF_LIB selects another build of the same ABI (A/B timing of kernel variants)
LIB_PATH = os.environ.get("IBF_LIB") or os.path.join(HERE, "libibf.so")

IBF_OK, IBF_ERR_BAD_ARG, IBF_ERR_CUDA, IBF_ERR_OOM, IBF_ERR_NONFINITE, IBF_ERR_NO_DEVICE, IBF_ERR_IO = range(7)
MODELS = {"snh": 0, "nh": 1, "cor": 2, "lin": 3}

_vp = C.c_void_p
_i64 = C.c_int64
_int = C.c_int
_dbl = C.c_double
_pi64 = C.POINTER(C.c_int64)
_pdbl = C.POINTER(C.c_double)

# name: (restype, argtypes)
_PROTOS = {
    "ibf_version": (C.c_char_p, []),
    "ibf_last_error": (C.c_char_p, []),
    "ibf_pair_eval": (_int, [_int, _i64, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ibf_accd": (_int, [_int, _i64, _vp, _vp, _dbl, _vp, _vp]),
    "ibf_ccd_create": (_int, [_i64, _vp, _i64, _vp, _i64, _vp, C.POINTER(_vp)]),
    "ibf_ccd_destroy": (None, [_vp]),
    "ibf_ccd_candidates": (_int, [_vp, _vp, _vp, _dbl, _pi64, _pi64, _vp]),
    "ibf_ccd_get_candidates": (_int, [_vp, _vp, _vp, _vp]),
    "ibf_max_step_size": (_int, [_vp, _vp, _vp, _dbl, _dbl, _pdbl, _pi64, _vp]),
    "ibf_ccd_get_blocking": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ibf_static_intersection": (_int, [_vp, _vp, _pi64, _vp, _i64, _vp]),
    "ibf_surface_extract": (_int, [_i64, _vp, C.POINTER(_vp), _pi64, _pi64, _pi64, _pi64, _vp]),
    "ibf_surface_get": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ibf_surface_destroy": (None, [_vp]),
    "ibf_export_obj": (_int, [C.c_char_p, _vp, _i64, _vp, _i64, _int]),
    "ibf_friction_create": (_int, [C.POINTER(_vp)]),
    "ibf_friction_destroy": (None, [_vp]),
    "ibf_friction_size": (_i64, [_vp]),
    "ibf_friction_precompute": (_int, [_vp, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _dbl, _pi64, _vp]),
    "ibf_friction_import": (_int, [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _dbl, _vp]),
    "ibf_friction_export": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _pdbl, _vp]),
    "ibf_system_set_friction": (_int, [_vp, _vp]),
    "ibf_min_distance": (_int, [_vp, _vp, _dbl, _pdbl, _vp, _vp]),
    "ibf_contacts_create": (_int, [_i64, _int, C.POINTER(_vp)]),
    "ibf_contacts_destroy": (None, [_vp]),
    "ibf_contacts_size": (_i64, [_vp]),
    "ibf_contacts_update": (_int, [_vp, _vp, _pi64, _pi64, _vp]),
    "ibf_contacts_update_host": (_int, [_vp, _i64, _vp, _vp, _vp, _pi64, _pi64, _vp]),
    "ibf_contacts_refresh_anchors": (_int, [_vp, _vp, _pi64, _vp]),
    "ibf_contacts_dual_sweep": (_int, [_vp, _vp, _dbl, _dbl, _dbl, _pdbl, _vp]),
    "ibf_contacts_export": (_int, [_vp] + [_vp] * 8 + [_vp]),
    "ibf_contacts_import": (_int, [_vp, _i64] + [_vp] * 8 + [_vp]),
    "ibf_system_create": (_int, [_i64, _vp, _vp, _int, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_vp)]),
    "ibf_system_destroy": (None, [_vp]),
    "ibf_system_pattern": (_int, [_vp, _pi64, _pi64]),
    "ibf_assemble": (_int, [_vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _int, _vp, _vp]),
    "ibf_system_matvec": (_int, [_vp, _vp, _vp, _vp]),
    "ibf_system_export_bsr": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ibf_system_pcg": (_int, [_vp, _vp, _vp, _dbl, _i64, _vp, _vp]),
    "ibf_incremental_energy": (_int, [_vp, _vp, _vp, _vp, _int, _vp, _vp, _dbl, _dbl, _dbl, _vp, _vp]),
    "ibf_inversion_safe_step": (_int, [_vp, _vp, _vp, _pdbl, _vp]),
    "ibf_stiffness_diagonal_max": (_int, [_vp, _vp, _dbl, _pdbl, _vp]),
    "ibf_solve_subproblem": (_int, [_vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _dbl, _vp, _vp]),
    "ibf_inertia_target": (_int, [_i64, _vp, _vp, _dbl, _vp, _vp, _vp]),
    "ibf_clamp_state": (_int, [_i64, _vp, _vp, _dbl, _vp]),
    "ibf_outer_loop": (_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _dbl, _dbl, _dbl, _int, _int,
                              _vp, _vp, _vp]),
    "ibf_velocity_update": (_int, [_i64, _vp, _vp, _dbl, _vp, _vp]),
    "ibf_bsr_create": (_int, [_i64, _i64, _vp, _vp, _vp, C.POINTER(_vp)]),
    "ibf_bsr_destroy": (None, [_vp]),
    "ibf_bsr_matvec": (_int, [_vp, _vp, _vp, _vp]),
    "ibf_bsr_mask_dirichlet": (_int, [_vp, _vp, _vp, _vp]),
    "ibf_bsr_pcg": (_int, [_vp, _vp, _vp, _dbl, _i64, _vp, _vp]),
    "ibf_system_spmv_stats": (_int, [_vp, _pdbl]),
    "ibf_bsr_size": (_i64, [_vp]),
    "ibf_vec_sub": (_int, [_i64, _vp, _vp, _vp, _vp]),
    "ibf_system_stats": (_int, [_vp, _vp, _int]),
    "ibf_ccd_stats": (_int, [_vp, _vp, _int]),
    "ibf_launch_count": (C.c_ulonglong, []),
    "ibf_bsr_export": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "ibf_pcg_tuning": (_int, [_i64, _int]),
    "ibf_dist_unique_id": (_int, [_vp]),
    "ibf_dist_create": (_int, [_int, _int, _vp, C.POINTER(_vp)]),
    "ibf_dist_create_local": (_int, [_int, C.POINTER(_vp)]),
    "ibf_dist_destroy": (None, [_vp]),
    "ibf_system_set_dist": (_int, [_vp, _vp]),
    "ibf_pcg_last_shape": (_int, [_vp]),
    "ibf_kernel_clocks": (_int, [_int, _vp, _int]),
    "ibf_system_counts": (_int, [_vp, _vp, _int]),
    "ibf_system_export_terms": (_int, [_vp, _pi64, _vp, _vp, _vp, _vp]),
}

_lib = None


class IbfError(RuntimeError):
    """A libibf call failed (CUDA error, bad argument, out of memory)."""


def lib():
    """Load libibf.so once; raises if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2512_12151_b200.build` "
                "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _PROTOS.items():
            if os.environ.get("IBF_LIB") and not hasattr(h, name):
                continue     # an older A/B build without this entry point
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols():
    return list(_PROTOS)


def check(status, what=""):
    if status == IBF_OK:
        return
    msg = lib().ibf_last_error().decode(errors="replace")
    if status == IBF_ERR_NONFINITE:
        from .solver import NonFiniteEnergyError
        raise NonFiniteEnergyError(msg)
    if status == IBF_ERR_BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    if status == IBF_ERR_IO:
        raise OSError(f"{what}: {msg}")
    raise IbfError(f"{what}: status {status}: {msg}")


def host_ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def dev_ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def stream():
    import torch
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


KERNEL_CLOCKS = ("k_elem", "k_gather_blocks", "k_vertex_rows", "k_energy", "k_traverse", "k_pair_toi", "k_pcg",
                 "k_prefilter", "k_refit")


def kernel_clocks(on=-1, reset=False):
    """{kernel: {ms, launches, bytes, flops, units}} from ibf_kernel_clocks."""
    out = np.zeros(5 * len(KERNEL_CLOCKS))
    check(lib().ibf_kernel_clocks(int(on), host_ptr(out), 1 if reset else 0), "ibf_kernel_clocks")
    return {k: dict(zip(("ms", "launches", "bytes", "flops", "units"), out[5 * i:5 * i + 5].tolist()))
            for i, k in enumerate(KERNEL_CLOCKS)}


def pcg_last_shape():
    """(ctas, threads, sweeps per thread, lanes per row, ready counter, terms)
    of the last PCG launch."""
    out = np.zeros(6, dtype=np.int64)
    check(lib().ibf_pcg_last_shape(host_ptr(out)), "ibf_pcg_last_shape")
    return tuple(int(v) for v in out)


class pcg_tuning:
    """Context manager over ibf_pcg_tuning: PCG launch-shape overrides for
    the solves inside the block (lanes_max_n 0 forces one thread per row;
    max_ctas caps the cooperative grid so each thread sweeps several rows)."""

    def __init__(self, lanes_max_n=-1, max_ctas=0):
        self.args = (int(lanes_max_n), int(max_ctas))

    def __enter__(self):
        check(lib().ibf_pcg_tuning(*self.args), "ibf_pcg_tuning")
        return self

    def __exit__(self, *exc):
        lib().ibf_pcg_tuning(-1, 0)
