"""ctypes loader for libgroot_b200.so (the C ABI declared in include/groot.h).

The product has no CPU fallback: if the library is missing or no CUDA device is
present, calls fail loudly with ``GrootError``.
"""
from __future__ import annotations

import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GROOT_LIB") or os.path.join(_PKG, "libgroot_b200.so")  # GROOT_LIB: experiment variant
_LIB = None

P = C.c_void_p
u8p = C.POINTER(C.c_uint8)
u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double

GROOT_OK, GROOT_EINVAL, GROOT_ERUNTIME, GROOT_ECUDA, GROOT_ENCCL = 0, 1, 2, 3, 4


class GrootError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class GrootInvalidArgument(GrootError, ValueError):
    """Raised where the reference throws std::invalid_argument."""


_SIG = {
    "groot_last_error": (C.c_char_p, []),
    "groot_version": (i32, []),
    "groot_set_stream": (i32, [P]),
    "groot_get_stream": (P, []),
    "groot_device_synchronize": (i32, []),
    "groot_kernel_launches": (u64, []),
    "groot_reset_kernel_launches": (None, []),
    "groot_profile_enable": (i32, [i32]),
    "groot_profile_read": (i32, [u32, P, P, P, P]),
    "groot_empty_cache": (i32, []),
    "groot_csa_sizes": (i32, [u32, P, P, P]),
    "groot_gen_csa": (i32, [u32, P, P, P]),
    "groot_csa_supports": (i32, [u32, P, P]),
    "groot_booth_sizes": (i32, [u32, P, P, P]),
    "groot_gen_booth": (i32, [u32, P, P, P]),
    "groot_aiger_sizes": (i32, [C.c_char_p, C.c_size_t, P, P, P]),
    "groot_aiger_fill": (i32, [C.c_char_p, C.c_size_t, P, P]),
    "groot_encode": (i32, [u32, u32, P, u32, P, P, P]),
    "groot_batch": (i32, [P, u32, P]),
    "groot_graph_from_host": (i32, [u32, P, P, P, P, u64, P, P]),
    "groot_graph_from_edges": (i32, [u32, P, P, u64, P, P]),
    "groot_graph_sizes": (i32, [P, P, P, P]),
    "groot_graph_copy_out": (i32, [P, P, P, P, P, P, P]),
    "groot_graph_device_ptrs": (i32, [P, P, P, P, P, P]),
    "groot_graph_free": (None, [P]),
    "groot_partition_topo_chunks": (i32, [P, u32, P]),
    "groot_partition_multilevel": (i32, [P, u32, u64, P, P, P]),
    "groot_load_assignment": (i32, [C.c_char_p, u32, P]),
    "groot_assignment_from_host": (i32, [u32, P, P]),
    "groot_assignment_info": (i32, [P, P, P]),
    "groot_assignment_copy_out": (i32, [P, P]),
    "groot_assignment_free": (None, [P]),
    "groot_crossing_fraction": (i32, [P, P, P]),
    "groot_edge_cut": (i32, [P, P, P]),
    "groot_regrow": (i32, [P, P, i32, P]),
    "groot_parts_count": (i32, [P, P]),
    "groot_parts_sizes": (i32, [P, u32, P, P, P]),
    "groot_parts_copy_out": (i32, [P, u32, P, P, P]),
    "groot_footprint_proxy": (i32, [P, u32, u32, P]),
    "groot_materialize": (i32, [P, P, u32, P]),
    "groot_parts_from_host": (i32, [u32, u32, P, P, P, P, P, P, P]),
    "groot_parts_free": (None, [P]),
    "groot_graph_prepare": (i32, [P]),
    "groot_graph_release_context": (i32, [P]),
    "groot_param_count": (u64, [u32, u32, u32, u32]),
    "groot_init_params": (i32, [u64, u32, u32, u32, u32, P]),
    "groot_model_create": (i32, [u32, u32, u32, u32, P, P]),
    "groot_model_load": (i32, [C.c_char_p, P]),
    "groot_model_save": (i32, [P, C.c_char_p]),
    "groot_model_info": (i32, [P, P, P, P, P]),
    "groot_model_params": (i32, [P, P]),
    "groot_model_free": (None, [P]),
    "groot_train": (i32, [P, u32, u32, u32, u32, u32, dbl, u64, dbl, dbl, dbl, P, P, P, P]),
    "groot_loss_and_grads": (i32, [P, u32, u32, u32, u32, P, P, P]),
    "groot_forward": (i32, [P, P, P]),
    "groot_debug_forward_naive": (i32, [P, P, P, P]),
    "groot_predict_full": (i32, [P, P, P, P, P]),
    "groot_predict": (i32, [P, P, P, P, P, P]),
    "groot_predict_full_dev": (i32, [P, P, P, P, P]),
    "groot_layer_dev": (i32, [P, P, u32, P, P, P, P]),
    "groot_predict_parts": (i32, [P, P, P, P, u32, P]),
    "groot_classify_aig": (i32, [P, u32, u32, P, u32, P, P, u32, P, P, P]),
    "groot_build_plan": (i32, [P, u32, u32, u32, P, P, P, P, P, P]),
    "groot_backward_rewrite": (i32, [u32, u32, P, u32, P, P, u32, P, P, u32, u64, P, P, P, P]),
    "groot_backward_rewrite_residual": (C.c_char_p, []),
    "groot_truth_table_equiv": (i32, [u32, u32, P, u32, P, u32, P]),
    "groot_simulate": (i32, [u32, u32, P, u32, P, P, P]),
    "groot_spmm_mean": (i32, [P, P, u32, P]),
    "groot_spmm_mean_dev": (i32, [P, P, u32, P]),
    "groot_spmm_csr": (i32, [u32, u32, P, P, P, P, u32, u32, P]),
    "groot_spmm_csr_f64": (i32, [u32, u32, P, P, P, P, u32, u32, P]),
    "groot_build_plan_rows": (i32, [u32, P, u32, u32, u32, P, P, P, P, P, P]),
    "groot_degree_sort": (i32, [u32, P, P, P]),
}

# Every symbol include/groot.h declares (checked by tests/test_capi.py).
EXPORTED = sorted(_SIG)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise GrootError(GROOT_ECUDA, f"{LIB_PATH} not built: run __graft_entry__.build() "
                                          "(no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIG.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int):
    if status != GROOT_OK:
        msg = lib().groot_last_error().decode()
        if status == GROOT_EINVAL:
            raise GrootInvalidArgument(status, msg)
        raise GrootError(status, msg)


def ptr(a):
    return None if a is None else C.c_void_p(a.ctypes.data)
