"""ctypes binding of the sm_100a shared library `_hdgb.so` (C ABI: include/hdgb.h).

The library is built in-tree by `paper_2007_11891_b200.build` (nvcc,
-gencode arch=compute_100a,code=sm_100a).  There is no CPU fallback: if the
library is missing or no CUDA device is visible, every device entry point
raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HDGB_LIB") or os.path.join(_HERE, "_hdgb.so")  # HDGB_LIB: tuning side builds

OK, EINVAL, EBREAKDOWN, ECUDA, ENCCL, ENONFINITE = 0, 1, 2, 3, 4, 5
INTERIOR, DIRICHLET, NEUMANN, HALO_OWNED, HALO_PEER = 0, 1, 2, 3, 4
PLAIN, TRANSFORMED = 0, 1
PREC_NONE, PREC_BLOCK, PREC_DIAG_NODAL, PREC_DIAG_EIGEN = 0, 1, 2, 3

_dp = ctypes.POINTER(ctypes.c_double)


class Desc(ctypes.Structure):
    _fields_ = [
        ("n_el", ctypes.c_int32 * 3),
        ("p", ctypes.c_int32),
        ("lam", ctypes.c_double),
        ("widths", _dp * 3),
        ("side_kind", ctypes.c_int32 * 6),
        ("S", _dp),
        ("B_S", _dp),
        ("Lambda", _dp),
        ("weights", _dp),
        ("GCC_diag", _dp),
        ("dz_inv", _dp),
        ("device", ctypes.c_int32),
    ]


# name -> (restype, argtypes); every symbol declared in include/hdgb.h
_VP = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
SIGNATURES = {
    "hdgb_last_error": (ctypes.c_char_p, []),
    "hdgb_version": (ctypes.c_char_p, []),
    "hdgb_ctx_create": (ctypes.c_int, [ctypes.POINTER(Desc), ctypes.POINTER(_VP)]),
    "hdgb_ctx_destroy": (ctypes.c_int, [_VP]),
    "hdgb_ctx_n_all": (_I64, [_VP]),
    "hdgb_ctx_n_unknown": (_I64, [_VP]),
    "hdgb_ctx_n_faces": (_I64, [_VP, ctypes.c_int]),
    "hdgb_op_apply": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP]),
    "hdgb_op_apply_host": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP]),
    "hdgb_op_apply_host_packed": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP]),
    "hdgb_face_transform": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "hdgb_prec_apply": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP, _VP]),
    "hdgb_diag_apply": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "hdgb_prec_table": (ctypes.c_int, [_VP, ctypes.c_int, _VP, _VP]),
    "hdgb_pack": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
    "hdgb_unpack": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
    "hdgb_zero_dirichlet": (ctypes.c_int, [_VP, _VP, _VP]),
    "hdgb_pcg": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, _VP, _VP, _D, _D, _I32,
                               ctypes.POINTER(_I32), ctypes.POINTER(_D), ctypes.POINTER(_I32), _VP]),
    "hdgb_dot_scratch_doubles": (_I64, []),
    "hdgb_vec_dot": (ctypes.c_int, [_VP, _VP, _I64, _VP, _VP, _VP]),
    "hdgb_ctx_set_element_tables": (ctypes.c_int, [_VP, _VP, _VP, _VP, _D]),
    "hdgb_hybridize": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP]),
    "hdgb_build_rhs": (ctypes.c_int, [_VP, _VP, _VP, _VP]),
    "hdgb_recover_interior": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "hdgb_element_inverse": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "hdgb_face_dot": (ctypes.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "hdgb_vec_axpby": (ctypes.c_int, [_I64, _D, _VP, _D, _VP, _VP, _VP]),
    "hdgb_halo_pack": (ctypes.c_int, [_VP, _VP, ctypes.c_int, _VP, _VP]),
    "hdgb_halo_add": (ctypes.c_int, [_VP, _VP, ctypes.c_int, _VP, _VP]),
    "hdgb_ctx_launches": (_I64, [_VP]),
    "hdgb_ctx_flags": (ctypes.c_int, [_VP]),
    "hdgb_fp64_peak": (ctypes.c_int, [ctypes.POINTER(_D), _VP]),
    "hdgb_nccl_unique_id": (ctypes.c_int, [_VP]),
    "hdgb_slab_group_create": (ctypes.c_int, [ctypes.POINTER(_VP), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, _VP, ctypes.POINTER(_VP)]),
    "hdgb_slab_group_destroy": (ctypes.c_int, [_VP]),
    "hdgb_slab_exchange": (ctypes.c_int, [_VP, ctypes.POINTER(_VP), _VP]),
    "hdgb_slab_apply": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _VP]),
    "hdgb_slab_pcg": (ctypes.c_int, [_VP, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_VP), ctypes.POINTER(_VP), _D, _D,
                                     _I32, ctypes.POINTER(_I32), ctypes.POINTER(_D), ctypes.POINTER(_I32), _VP]),
}

_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load `_hdgb.so` once; raise loudly if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LibraryMissing(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the hot path)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("HDGB_LIB") and not hasattr(L, name):
                continue  # an older side build (A/B timing) may lack newer entry points
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status):
    """Map an hdgb_status to the reference's Python exceptions."""
    if status == OK:
        return
    msg = lib().hdgb_last_error().decode(errors="replace")
    if status == EINVAL:
        raise ValueError(msg)
    if status in (EBREAKDOWN, ENONFINITE):
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def dptr(arr):
    """ctypes double* of a contiguous float64 numpy array."""
    return arr.ctypes.data_as(_dp)
