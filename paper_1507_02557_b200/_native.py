"""ctypes binding of the C ABI in include/hybridwave_b200.h.

The product path has no CPU fallback: if the shared library is missing or
was built without the requested order, every entry point raises.
"""

import ctypes
import os
from ctypes import c_double, c_int, c_int32, c_int64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libhybridwave_b200.so"
LIB_PATH = os.path.join(_HERE, LIB_NAME)

HW_HEX, HW_WEDGE, HW_PYRAMID, HW_TET = 0, 1, 2, 3
HW_F64, HW_F32 = 0, 1
HW_FORM_STRONG, HW_FORM_SKEW = 0, 1
HW_GL, HW_SEM = 0, 1
HW_NBR_BOUNDARY = 0x200


class HWType(ctypes.Structure):
    _fields_ = [("K", c_int64), ("geo", c_void_p), ("mat", c_void_p),
                ("nbr_elem", c_void_p), ("nbr_code", c_void_p),
                ("op", c_void_p * 10), ("iop", c_void_p * 4),
                ("form", c_int32), ("pad_", c_int32)]


class HWMesh(ctypes.Structure):
    _fields_ = [("N", c_int32), ("dtype", c_int32), ("formulation", c_int32),
                ("device", c_int32), ("penalty_scale", c_double),
                ("perm_tri", c_void_p), ("perm_quad", c_void_p),
                ("tr_in", c_void_p * 4), ("tr_out", c_void_p * 4),
                ("t", HWType * 4), ("frc", c_void_p * 4)]


class HWFields(ctypes.Structure):
    _fields_ = [("p", c_void_p * 4)]


class HWSubset(ctypes.Structure):
    _fields_ = [("idx", c_void_p * 4), ("n", c_int64 * 4)]


class NativeError(RuntimeError):
    pass


_lib = None


def lib():
    """Load the in-tree library once; raise loudly if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (nvcc, sm_100a). "
                "There is no CPU fallback for the hot path.")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        L.hw_rhs.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWSubset), c_void_p]
        L.hw_traces.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWSubset), c_void_p]
        L.hw_lsrk_stage.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWFields),
                                    c_double, c_double, c_double, P(HWSubset), c_void_p]
        L.hw_ab_step.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWFields),
                                 P(HWFields), P(HWFields), c_int, c_double, c_double,
                                 c_double, c_double, P(HWSubset), c_void_p]
        L.hw_axpy3.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWFields),
                               P(HWFields), P(HWFields), c_int, c_double, c_double,
                               c_double, c_double, P(HWSubset), c_void_p]
        L.hw_hist_push.argtypes = [P(HWMesh), P(HWFields), P(HWFields), P(HWFields),
                                   P(HWFields), P(HWSubset), c_void_p]
        L.hw_halo_pack.argtypes = [P(HWMesh), c_int, c_void_p, c_void_p, c_int64,
                                   c_void_p, c_void_p]
        L.hw_energy.argtypes = [P(HWMesh), P(HWFields), c_void_p, c_void_p]
        L.hw_forcing.argtypes = [P(HWMesh), c_int, c_void_p, c_void_p, c_void_p, c_void_p,
                                 c_int, c_double, c_void_p, c_double, c_void_p, c_int,
                                 c_void_p]
        L.hw_wedge_face_correction.argtypes = [P(HWMesh), c_int, c_int, c_void_p, c_void_p,
                                               c_void_p, c_void_p, c_int, c_int, c_void_p,
                                               c_void_p]
        L.hw_prepare.argtypes = [P(HWMesh)]
        L.hw_halo_gather.argtypes = [P(HWMesh), c_void_p, c_int64, c_void_p, c_int64,
                                     c_void_p, c_void_p]
        L.hw_halo_scatter.argtypes = [P(HWMesh), c_void_p, c_int64, c_void_p, c_int64,
                                      c_void_p, c_void_p]
        L.hw_last_error.restype = ctypes.c_char_p
        for name in ("hw_rhs", "hw_traces", "hw_lsrk_stage", "hw_ab_step", "hw_axpy3",
                     "hw_hist_push", "hw_halo_pack", "hw_halo_gather", "hw_halo_scatter",
                     "hw_forcing", "hw_wedge_face_correction", "hw_prepare", "hw_energy", "hw_version", "hw_supported_orders"):
            getattr(L, name).restype = c_int
        L.hw_launch_count.restype = ctypes.c_longlong
        L.hw_launch_count.argtypes = []
        _lib = L
    return _lib


EXPORTED_SYMBOLS = ("hw_rhs", "hw_traces", "hw_lsrk_stage", "hw_ab_step", "hw_axpy3", "hw_hist_push",
                    "hw_halo_pack", "hw_halo_gather", "hw_halo_scatter", "hw_forcing",
                    "hw_wedge_face_correction", "hw_prepare", "hw_energy", "hw_last_error", "hw_version",
                    "hw_supported_orders", "hw_launch_count")


def check(rc):
    if rc != 0:
        raise ValueError(f"hybridwave_b200: {lib().hw_last_error().decode()}")


def fields(tensors):
    """HWFields from a 4-slot list of torch tensors / None."""
    f = HWFields()
    for i, t in enumerate(tensors):
        f.p[i] = None if t is None else t.data_ptr()
    return f


def subset(lists):
    """HWSubset from a 4-slot list of int32 device tensors (None = all)."""
    s = HWSubset()
    for i, t in enumerate(lists):
        if t is None:
            s.idx[i] = None
            s.n[i] = -1
        else:
            s.idx[i] = t.data_ptr()
            s.n[i] = t.numel()
    return s
