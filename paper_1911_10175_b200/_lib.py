"""ctypes binding of ``libspconv_b200.so`` (the C ABI in include/spconv_b200.h).

There is no fallback: if the shared library is missing the import fails with
an error telling you to build it, and every pass returns SPC_ERR_NO_DEVICE
(raised as SpconvError) when no B200 is visible.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# SPC_LIB_PATH: alternative build of the same library (A/B timing in tools/)
LIB_PATH = os.environ.get("SPC_LIB_PATH") or os.path.join(HERE, "libspconv_b200.so")

SPC_OK, SPC_ERR_SHAPE, SPC_ERR_PLAN, SPC_ERR_LAYOUT, SPC_ERR_ARG, SPC_ERR_CUDA, SPC_ERR_NCCL, SPC_ERR_NO_DEVICE = range(8)
STATUS_NAMES = {0: "SPC_OK", 1: "SPC_ERR_SHAPE", 2: "SPC_ERR_PLAN", 3: "SPC_ERR_LAYOUT", 4: "SPC_ERR_ARG",
                5: "SPC_ERR_CUDA", 6: "SPC_ERR_NCCL", 7: "SPC_ERR_NO_DEVICE"}


class spc_shape(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "C", "K", "H", "W", "R", "S", "O", "P", "padW", "padH")]


class spc_plan(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("comp", "check", "V", "Q", "T", "pipelined", "ring_size", "M",
                                        "register_budget", "unroll_hint", "prefetch_hints")]


class spc_epilogue(C.Structure):
    _fields_ = [("alpha", C.c_float), ("add", C.c_void_p), ("mask", C.c_void_p), ("relu", C.c_int),
                ("beta", C.c_float)]


class spc_counters(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("checked_vectors", "executed_vector_fmas",
                                           "output_vector_loads", "output_vector_stores")]


class spc_tensor(C.Structure):
    _fields_ = [("layout", C.c_int), ("V", C.c_int), ("n", C.c_int), ("c", C.c_int), ("h", C.c_int),
                ("w", C.c_int), ("k", C.c_int), ("r", C.c_int), ("s", C.c_int),
                ("data", C.c_void_p), ("numel", C.c_size_t)]


class spc_host_pass(C.Structure):
    _fields_ = [("a", C.POINTER(spc_tensor)), ("b", C.POINTER(spc_tensor)), ("shape", C.POINTER(spc_shape)),
                ("plan", C.POINTER(spc_plan)), ("mode", C.c_int), ("dst", C.POINTER(spc_tensor)),
                ("counters", C.POINTER(spc_counters)), ("status", C.c_int), ("flags", C.c_int)]


SPC_PASS_CHECKED_NCHWC = 1


# name -> (restype, argtypes)
_SIGS = {
    "spc_abi_version": (C.c_int, []),
    "spc_last_error": (C.c_char_p, []),
    "spc_backend_name": (C.c_char_p, []),
    "spc_native_backend_available": (C.c_int, [C.c_int]),
    "spc_launch_count": (C.c_uint64, []),
    "spc_set_math": (C.c_int, [C.c_int]),
    "spc_get_math": (C.c_int, []),
    "spc_shape_make": (C.c_int, [C.c_int] * 9 + [C.POINTER(spc_shape)]),
    "spc_shape_make_padded": (C.c_int, [C.c_int] * 11 + [C.POINTER(spc_shape)]),
    "spc_shape_validate": (C.c_int, [C.POINTER(spc_shape)]),
    "spc_plan_make": (C.c_int, [C.POINTER(spc_shape), C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(spc_plan)]),
    "spc_output_desc": (C.c_int, [C.POINTER(spc_shape), C.POINTER(spc_plan), C.POINTER(spc_tensor)]),
    "spc_analytic_counters": (C.c_int, [C.POINTER(spc_shape), C.POINTER(spc_plan), C.c_int,
                                        C.POINTER(spc_counters)]),
    "spc_sparse_fwd": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                 C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p, C.c_void_p]),
    "spc_sparse_bwi": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                 C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p, C.c_void_p]),
    "spc_sparse_bww": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                 C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p, C.c_void_p]),
    "spc_run_parallel": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                   C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p, C.c_void_p]),
    "spc_sparse_fwd_ex": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                    C.POINTER(spc_plan), C.c_int, C.POINTER(spc_epilogue), C.POINTER(spc_tensor),
                                    C.c_void_p, C.c_void_p]),
    "spc_sparse_bwi_ex": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                    C.POINTER(spc_plan), C.c_int, C.POINTER(spc_epilogue), C.POINTER(spc_tensor),
                                    C.c_void_p, C.c_void_p]),
    "spc_epilogue_apply": (C.c_int, [C.POINTER(spc_epilogue), C.c_void_p, C.c_size_t, C.c_void_p]),
    "spc_run_parallel_host": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                        C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor),
                                        C.POINTER(spc_counters)]),
    "spc_run_parallel_host_batch": (C.c_int, [C.POINTER(spc_host_pass), C.c_int]),
    "spc_host_batch_release": (None, []),
    "spc_relu": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "spc_relu_grad_mask": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "spc_nchwc_to_chwnn": (C.c_int, [C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.c_void_p]),
    "spc_ffma_peak_kernel": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double), C.c_void_p]),
    "spc_l2_flush": (C.c_int, [C.c_void_p, C.c_size_t, C.c_void_p]),
    "spc_gen_sparse": (C.c_int, [C.c_void_p, C.c_size_t, C.c_double, C.c_uint64]),
    "spc_vector_probe": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_float, C.c_void_p,
                                   C.POINTER(C.c_uint32)]),
    # multi-GPU: batch-sharded BWW exchange (csrc/comm.cu)
    "spc_nccl_version": (C.c_int, []),
    "spc_comm_unique_id": (C.c_int, [C.c_void_p]),
    "spc_comm_init": (C.c_int, [C.POINTER(C.c_void_p), C.c_int, C.c_void_p, C.c_int]),
    "spc_comm_wrap": (C.c_int, [C.POINTER(C.c_void_p), C.c_void_p]),
    "spc_comm_nccl": (C.c_void_p, [C.c_void_p]),
    "spc_comm_size": (C.c_int, [C.c_void_p]),
    "spc_comm_rank": (C.c_int, [C.c_void_p]),
    "spc_comm_destroy": (C.c_int, [C.c_void_p]),
    "spc_comm_window_alloc": (C.c_int, [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(C.c_int)]),
    "spc_comm_window_free": (C.c_int, [C.c_void_p, C.c_void_p]),
    "spc_bww_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]),
    "spc_bww_sharded": (C.c_int, [C.c_void_p, C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                  C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p, C.c_void_p]),
}

# Every symbol include/spconv_b200.h declares (checked by the CPU test suite).
EXPORTED = tuple(_SIGS)

# include/spconv_b200_dev.h (development entry points)
_DEV_SIGS = {
    "spc_debug_conv_variant": (C.c_int, [C.c_int, C.POINTER(spc_tensor), C.POINTER(spc_tensor), C.POINTER(spc_shape),
                                         C.POINTER(spc_plan), C.c_int, C.POINTER(spc_tensor), C.c_void_p,
                                         C.c_void_p]),
}
DEV_EXPORTED = tuple(_DEV_SIGS)

_lib = None


def load():
    """Load the product library; raises ImportError if it was never built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build the CUDA library first "
                "(python -c 'import __graft_entry__ as g; g.build()'). There is no CPU fallback.")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in {**_SIGS, **_DEV_SIGS}.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        if L.spc_abi_version() != 3:
            raise ImportError("libspconv_b200.so ABI version mismatch")
        _lib = L
    return _lib


def last_error() -> str:
    return load().spc_last_error().decode()
