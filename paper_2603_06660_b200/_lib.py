"""ctypes binding of libpag_gpu.so (the C ABI in include/pag_gpu.h).

The native library is the product: there is no Python or CPU fallback.
Importing this module raises ImportError when the library is missing, and
every call raises when it fails.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAG_GPU_LIB") or os.path.join(HERE, "libpag_gpu.so")

PAG_GPU_OK = 0
PAG_GPU_EINVAL = 1
PAG_GPU_ERUNTIME = 2
PAG_GPU_ELOGIC = 3
PAG_GPU_ENOMEM = 4
PAG_GPU_ECUDA = 5

# the exported symbol set declared by include/pag_gpu.h
EXPORTS = (
    "pag_gpu_default_params",
    "pag_gpu_open",
    "pag_gpu_open_devices",
    "pag_gpu_open_from_arrays",
    "pag_gpu_refresh_from_arrays",
    "pag_gpu_close",
    "pag_gpu_info",
    "pag_gpu_search",
    "pag_gpu_search_device",
    "pag_gpu_search_submit",
    "pag_gpu_search_wait",
    "pag_gpu_construction_search",
    "pag_gpu_construction_submit",
    "pag_gpu_construction_search_device",
    "pag_gpu_ground_truth",
    "pag_gpu_refresh",
    "pag_gpu_inspect",
    "pag_gpu_reference_family",
    "pag_gpu_default_subspace_count",
    "pag_gpu_last_error",
    "pag_gpu_version",
)


class SearchStatsC(C.Structure):
    _fields_ = [("exact_dist_count", C.c_uint64), ("test_count", C.c_uint64),
                ("pass_count", C.c_uint64), ("visited_count", C.c_uint64),
                ("edges_scanned", C.c_uint64)]


class SearchParamsC(C.Structure):
    _fields_ = [("K", C.c_uint32), ("efS", C.c_uint32), ("b_override", C.c_uint32),
                ("use_prt", C.c_uint8), ("use_tfb", C.c_uint8), ("exact_dist", C.c_uint8),
                ("reserved", C.c_uint8)]


class IndexArraysC(C.Structure):
    """pag_index_arrays: the reference's in-memory PagIndex, borrowed for a call."""
    _fields_ = [("n", C.c_uint64), ("dim", C.c_uint32), ("padded_dim", C.c_uint32), ("L", C.c_uint32),
                ("m", C.c_uint32), ("M", C.c_uint32), ("efC", C.c_uint32), ("b_build", C.c_uint32),
                ("pes_flush_interval", C.c_uint32), ("seed", C.c_uint64), ("metric", C.c_uint8),
                ("enable_pes", C.c_uint8), ("reserved", C.c_uint8 * 2), ("n_entries", C.c_uint32),
                ("entry_nodes", C.c_void_p), ("degrees", C.c_void_p), ("targets", C.c_void_p),
                ("scalars", C.c_void_p), ("codes", C.c_void_p), ("rows", C.c_void_p), ("norms", C.c_void_p)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python __graft_entry__.py` or "
            "`make -C paper_2603_06660_b200/csrc` (no CPU fallback exists)")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
    u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
    sig = {
        "pag_gpu_default_params": (None, [C.POINTER(SearchParamsC)]),
        "pag_gpu_open": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(P)]),
        "pag_gpu_open_devices": (C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.c_uint32, C.POINTER(P)]),
        "pag_gpu_open_from_arrays": (C.c_int, [C.POINTER(IndexArraysC), C.POINTER(C.c_int), C.c_uint32,
                                               C.POINTER(P)]),
        "pag_gpu_refresh_from_arrays": (C.c_int, [P, C.POINTER(IndexArraysC), u64p]),
        "pag_gpu_close": (C.c_int, [P]),
        "pag_gpu_info": (C.c_int, [P, u64p, C.c_size_t]),
        "pag_gpu_search": (C.c_int, [P, C.c_void_p, C.c_uint64, C.POINTER(SearchParamsC),
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "pag_gpu_search_device": (C.c_int, [P, C.c_void_p, C.c_uint64, C.POINTER(SearchParamsC),
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p]),
        "pag_gpu_search_submit": (C.c_int, [P, C.c_void_p, C.c_uint64, C.POINTER(SearchParamsC),
                                            C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.POINTER(C.c_uint64)]),
        "pag_gpu_search_wait": (C.c_int, [P, C.c_uint64]),
        "pag_gpu_construction_search": (C.c_int, [P, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p, C.c_uint32, C.c_void_p]),
        "pag_gpu_construction_submit": (C.c_int, [P, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p, C.c_uint32, C.c_void_p, C.POINTER(C.c_uint64)]),
        "pag_gpu_construction_search_device": (C.c_int, [P, C.c_void_p, C.c_uint64, C.c_void_p, C.c_int,
                                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                         C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
        "pag_gpu_ground_truth": (C.c_int, [P, f32p, C.c_uint64, C.c_uint32, u32p, f32p]),
        "pag_gpu_refresh": (C.c_int, [P, C.c_char_p, u64p]),
        "pag_gpu_inspect": (C.c_int, [C.c_char_p, u64p, C.c_size_t]),
        "pag_gpu_reference_family": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, f32p,
                                               C.c_size_t]),
        "pag_gpu_default_subspace_count": (C.c_uint32, [C.c_uint32]),
        "pag_gpu_last_error": (C.c_char_p, []),
        "pag_gpu_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()


class PagGpuError(RuntimeError):
    """A CUDA-side failure (no reference counterpart)."""


def check(rc: int) -> None:
    if rc == PAG_GPU_OK:
        return
    msg = lib.pag_gpu_last_error().decode()
    if rc == PAG_GPU_EINVAL:
        raise ValueError(msg)          # std::invalid_argument
    if rc == PAG_GPU_ELOGIC:
        raise AssertionError(msg)      # std::logic_error
    if rc == PAG_GPU_ENOMEM:
        raise MemoryError(msg)
    if rc == PAG_GPU_ECUDA:
        raise PagGpuError(msg)
    raise RuntimeError(msg)            # std::runtime_error
