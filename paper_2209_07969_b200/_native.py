"""ctypes binding of the C-ABI in ``include/pf_b200.h`` (``libpfb200.so``).

The library is built in-tree by ``paper_2209_07969_b200.build.build()`` (nvcc, sm_100a).  There
is deliberately no fallback: if the shared object is missing, importing the solver fails loudly.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PFB200_LIB") or os.path.join(HERE, "libpfb200.so")

PF_OK, PF_ERR_INVALID, PF_ERR_INDEX = 0, 1, 2
PF_ERR_CONV_MOMENTUM, PF_ERR_CONV_EVOLUTION, PF_ERR_CONV_STAGGERED = 3, 4, 5
PF_ERR_SINGULAR, PF_ERR_CUDA, PF_ERR_NCCL = 6, 7, 8

SCHEME_CODES = {"ST": 0, "S1": 1, "S2": 2, "S3": 3}

_i32p = C.POINTER(C.c_int32)
_i64p = C.POINTER(C.c_int64)
_f64p = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class PfMesh(C.Structure):
    _fields_ = [
        ("nx", C.c_int32), ("ny", C.c_int32), ("hx", C.c_double), ("hy", C.c_double),
        ("node_lo", _i32p), ("node_hi", _i32p), ("node_start", _i64p),
        ("elem_lo", _i32p), ("elem_hi", _i32p), ("elem_start", _i64p),
        ("notch_row", C.c_int32), ("notch_lo", C.c_int32), ("notch_hi", C.c_int32),
        ("dup_start", C.c_int64), ("n_nodes", C.c_int64), ("n_elems", C.c_int64),
    ]


class PfMaterial(C.Structure):
    _fields_ = [
        ("mu", C.c_double), ("lam", C.c_double), ("bulk_k", C.c_double), ("g_c", C.c_double),
        ("length_l", C.c_double), ("eta", C.c_double), ("c_w", C.c_double),
        ("gamma", C.c_double), ("at2", C.c_int32),
    ]


class PfConfig(C.Structure):
    _fields_ = [
        ("tol_nr", C.c_double), ("tol_st", C.c_double), ("d_cap", C.c_double),
        ("res_floor", C.c_double), ("max_nr", C.c_int32), ("max_stag", C.c_int32),
        ("cg_rtol", C.c_double), ("cg_maxiter_factor", C.c_int32),
    ]


class PfStats(C.Structure):
    _fields_ = [
        ("n_stag", C.c_int32), ("n_nr_u", C.c_int32), ("n_nr_d", C.c_int32),
        ("spd_fallbacks", C.c_int32), ("final_rd_ratio", C.c_double),
        ("final_ru_ratio", C.c_double), ("wall_u", C.c_double), ("wall_d", C.c_double),
        ("n_hist", C.c_int32), ("cg_iters_u", C.c_int64), ("cg_iters_d", C.c_int64),
        ("cg_dofiters_u", C.c_double), ("cg_dofiters_d", C.c_double),
        ("kernel_ms_u", C.c_double), ("kernel_ms_d", C.c_double),
        ("cg_launches_u", C.c_int32), ("cg_launches_d", C.c_int32), ("launches", C.c_int32),
        ("step_ms", C.c_double),
    ]


class PfStrip(C.Structure):
    _fields_ = [
        ("rank", C.c_int32), ("nranks", C.c_int32),
        ("own_lo", C.c_int64), ("own_hi", C.c_int64), ("dup_lo", C.c_int64),
        ("cell_lo", C.c_int64), ("cell_hi", C.c_int64),
        ("send_lo_start", C.c_int64), ("send_lo_count", C.c_int64),
        ("recv_lo_start", C.c_int64), ("recv_lo_count", C.c_int64),
        ("send_hi_start", C.c_int64), ("send_hi_count", C.c_int64),
        ("recv_hi_start", C.c_int64), ("recv_hi_count", C.c_int64),
        ("comm_kind", C.c_int32), ("nccl_id", C.c_ubyte * 128), ("host_group", C.c_void_p),
    ]


# name -> (restype, argtypes); mirrors include/pf_b200.h
_SIGNATURES = {
    "pf_create": (C.c_int, [C.POINTER(PfMesh), C.POINTER(PfMaterial), C.POINTER(PfConfig),
                            C.c_int, C.POINTER(C.c_void_p)]),
    "pf_destroy": (None, [C.c_void_p]),
    "pf_last_error": (C.c_char_p, [C.c_void_p]),
    "pf_version": (C.c_char_p, []),
    "pf_set_state": (C.c_int, [C.c_void_p] + [_f64p] * 7),
    "pf_get_state": (C.c_int, [C.c_void_p] + [_f64p] * 7),
    "pf_get_gp_strain": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "pf_interp_nodal": (C.c_int, [C.c_void_p, _f64p, _f64p]),
    "pf_staggered_step": (C.c_int, [C.c_void_p, C.c_int, _i64p, _i64p, _f64p, C.c_int32,
                                    _i64p, C.c_int64, C.POINTER(PfStats), _f64p, C.c_int32]),
    "pf_solve_momentum": (C.c_int, [C.c_void_p, _i64p, _i64p, _f64p, C.c_int32, _f64p, _i32p,
                                    _f64p]),
    "pf_solve_evolution": (C.c_int, [C.c_void_p, C.c_int, _i64p, C.c_int64, _f64p, _i32p,
                                     _i32p]),
    "pf_evolution_residual_norm": (C.c_int, [C.c_void_p, _i64p, C.c_int64, _f64p]),
    "pf_commit_step": (C.c_int, [C.c_void_p]),
    "pf_internal_force": (C.c_int, [C.c_void_p, _f64p]),
    "pf_reaction_force": (C.c_int, [C.c_void_p, _i64p, C.c_int64, C.c_int, _f64p]),
    "pf_momentum_tangent_apply": (C.c_int, [C.c_void_p, _f64p, _f64p, _f64p]),
    "pf_evolution_residual": (C.c_int, [C.c_void_p, _f64p]),
    "pf_evolution_tangent_apply": (C.c_int, [C.c_void_p, C.c_int, _f64p, _f64p, _f64p]),
    "pf_refresh_gp": (C.c_int, [C.c_void_p]),
    "pf_softening_gate": (C.c_int, [C.c_void_p, _u8p]),
    "pf_extra_stiffness": (C.c_int, [C.c_void_p, C.c_int, _f64p]),
    "pf_update_active_energy": (C.c_int, [C.c_void_p, C.c_int, _f64p]),
    "pf_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte * 128)]),
    "pf_host_group_create": (C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    "pf_host_group_destroy": (None, [C.c_void_p]),
    "pf_create_strip": (C.c_int, [C.POINTER(PfMesh), C.POINTER(PfMaterial), C.POINTER(PfConfig),
                                  C.c_int, C.POINTER(PfStrip), C.POINTER(C.c_void_p)]),
    "pf_bench_mg_kernel": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _f64p, _f64p]),
    "pf_bench_cg": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, _f64p, _i64p]),
    "pf_device_info": (C.c_int, [C.c_void_p, _i32p, _i32p, _i64p]),
    "pf_host_alloc": (C.c_int, [C.c_int64, C.POINTER(C.c_void_p)]),
    "pf_host_free": (None, [C.c_void_p]),
    "pf_mg_info": (C.c_int, [C.c_void_p, _i32p, _i32p, _i32p, _i64p, _f64p]),
    "pf_solver_kinds": (C.c_int, [C.c_void_p, _i32p, _i32p]),
    "pf_init_state": (C.c_int, [C.c_void_p, _f64p, C.c_int64, C.c_double, C.c_double, C.c_double]),
    "pf_flush_l2": (C.c_int, [C.c_void_p]),
    "pf_synchronize": (C.c_int, [C.c_void_p]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def load():
    """Load ``libpfb200.so`` (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def f64(a):
    """Pointer to a C-contiguous float64 array (None -> NULL)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"], "expected contiguous float64"
    return a.ctypes.data_as(_f64p)


def i64(a):
    if a is None:
        return None
    assert a.dtype == np.int64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_i64p)


def i32(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_i32p)


def u8(a):
    assert a.dtype == np.uint8 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_u8p)


class PinnedPool:
    """Page-locked float64 arrays for the state outputs (pf_host_alloc): the device writes them
    by direct DMA.  A buffer returns to the pool when its array is garbage collected, so the
    drop-in's per-step output arrays (rebound like the reference's, schemes.py:391,
    assembly.py:265-269) cycle through two sets of buffers."""

    def __init__(self):
        self.free = {}

    def empty(self, shape):
        import weakref

        lib = load()
        n = int(np.prod(shape))
        nbytes = max(8 * n, 8)
        stack = self.free.setdefault(nbytes, [])
        if stack:
            ptr = stack.pop()
        else:
            p = C.c_void_p()
            if lib.pf_host_alloc(nbytes, C.byref(p)) != 0:
                return np.empty(shape)  # no pinned memory left: pageable (staged) output
            ptr = p.value
        buf = (C.c_char * nbytes).from_address(ptr)
        flat = np.frombuffer(buf, dtype=np.float64, count=n)
        # every view (reshape included) keeps `flat` alive: numpy collapses view bases to it
        weakref.finalize(flat, stack.append, ptr)
        return flat.reshape(shape)


PINNED = PinnedPool()
