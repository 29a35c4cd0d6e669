"""ctypes binding of the C ABI in include/anisoq_b200.h.

The library is built in-tree (paper_1908_10396_b200/libanisoq_b200.so, see
build.py). There is no fallback: if the shared library is missing or cannot
be loaded, importing the product path raises.
"""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libanisoq_b200.so")


class aq_weights(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("h_parallel", C.c_double),
        ("h_perpendicular", C.c_double),
        ("h_parallel_arr", C.c_void_p),
        ("h_perpendicular_arr", C.c_void_p),
        ("threshold", C.c_double),
        ("threshold_policy", C.c_int),
    ]


class aq_train_config(C.Structure):
    _fields_ = [
        ("max_iterations", C.c_int),
        ("relative_tolerance", C.c_double),
        ("seed", C.c_uint64),
        ("empty_partition_policy", C.c_int),
        ("ridge", C.c_double),
        ("threads", C.c_int),
        ("sweep_to_fixed_point", C.c_int),
    ]


_VP = C.c_void_p
_SZ = C.c_size_t
_I = C.c_int
_D = C.c_double
_PP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "aq_error_class": (_I, [_I]),
    "aq_last_error": (C.c_char_p, []),
    "aq_status_name": (C.c_char_p, [_I]),
    "aq_session_create": (_I, [_I, _PP]),
    "aq_session_destroy": (_I, [_VP]),
    "aq_session_stream": (_VP, [_VP]),
    "aq_session_sync": (_I, [_VP]),
    "aq_session_launches": (C.c_uint64, [_VP]),
    "aq_session_timing": (_I, [_VP, _I]),
    "aq_session_timer_read": (_I, [_VP, _I, _VP, _VP, _I]),
    "aq_dev_search_rerank_d": (_I, [_VP, _VP, _VP, _VP, _SZ, _SZ, _SZ, _VP, _VP, _VP, _VP]),
    "aq_dataset_upload": (_I, [_VP, _VP, _SZ, _SZ, _PP]),
    "aq_dataset_upload_f64": (_I, [_VP, _VP, _SZ, _SZ, _PP]),
    "aq_dataset_is_f64": (_I, [_VP]),
    "aq_dataset_wrap_device": (_I, [_VP, _VP, _SZ, _SZ, _PP]),
    "aq_dataset_free": (_I, [_VP]),
    "aq_dataset_norms": (_I, [_VP, _VP]),
    "aq_codebook_upload": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _PP]),
    "aq_codebook_download": (_I, [_VP, _VP]),
    "aq_codebook_free": (_I, [_VP]),
    "aq_codes_alloc": (_I, [_VP, _SZ, _SZ, _SZ, _PP]),
    "aq_codes_upload": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _PP]),
    "aq_codes_upload_packed": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _PP]),
    "aq_codes_download": (_I, [_VP, _VP]),
    "aq_codes_download_packed": (_I, [_VP, _VP]),
    "aq_codes_row_bytes": (_SZ, [_VP]),
    "aq_codes_free": (_I, [_VP]),
    "aq_dev_pq_quantize": (_I, [_VP, _VP, _VP, _I, _VP]),
    "aq_dev_pq_assign_pass": (_I, [_VP, _VP, _VP, _I, _VP, _VP, _VP]),
    "aq_pq_quantize": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _I, _VP]),
    "aq_pq_assign_pass": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _I, _VP, _VP]),
    "aq_pq_assign_point": (_I, [_VP, _VP, _SZ, _VP, _VP, _SZ, _SZ, _SZ, _D, _D, _VP]),
    "aq_pq_assign_point_order": (_I, [_VP, _VP, _SZ, _VP, _VP, _SZ, _SZ, _SZ, _D, _D, _VP, _SZ,
                                      _VP]),
    "aq_build_lut": (_I, [_VP, _VP, _SZ, _VP, _SZ, _SZ, _SZ, _VP]),
    "aq_dev_adc_search": (_I, [_VP, _VP, _VP, _SZ, _SZ, _VP, _VP]),
    "aq_dev_adc_search_d": (_I, [_VP, _VP, _VP, _SZ, _SZ, _VP, _VP]),
    "aq_dev_search_rerank": (_I, [_VP, _VP, _VP, _VP, _SZ, _SZ, _SZ, _VP, _VP, _VP, _VP]),
    "aq_dev_exact_dots_d": (_I, [_VP, _VP, _SZ, _VP, _SZ, _VP]),
    "aq_adc_search": (_I, [_VP, _VP, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _SZ,
                           _VP, _VP, _VP]),
    "aq_dev_rerank": (_I, [_VP, _VP, _SZ, _VP, _SZ, _SZ, _VP, _VP]),
    "aq_dev_exact_search": (_I, [_VP, _VP, _SZ, _SZ, _VP, _VP]),
    "aq_dev_assemble_selector_system": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "aq_dev_pq_codebook_update": (_I, [_VP, _VP, _VP, _D, _VP]),
    "aq_pq_codebook_update": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _VP, _D, _VP]),
    "aq_dev_train_l2_pq": (_I, [_VP, _SZ, _SZ, _VP, _PP, _PP]),
    "aq_debug_exact_window_count": (_I, [_VP, _I, _VP]),
    "aq_dev_train_apq": (_I, [_VP, _SZ, _SZ, _VP, _VP, _I, _PP, _PP, _VP, _VP]),
    "aq_dev_train_avq": (_I, [_VP, _SZ, _VP, _VP, _PP, _PP, _VP, _VP]),
    "aq_train_avq": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _VP, _VP, _VP, _VP, _VP, _VP]),
    # host-pointer forms
    "aq_adc_search_batch": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _SZ,
                                 _VP, _VP]),
    "aq_rerank": (_I, [_VP, _VP, _SZ, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _VP, _VP]),
    "aq_exact_search_batch": (_I, [_VP, _VP, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _VP]),
    "aq_assemble_selector_system": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _VP, _VP, _VP]),
    "aq_train_l2_pq": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _SZ, _VP, _VP, _VP]),
    "aq_train_apq": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _SZ, _VP, _VP, _I, _VP, _VP, _VP, _VP]),
    # multi-device session (csrc/multi.cu)
    "aq_device_count": (_I, [_VP]),
    "aq_multi_create": (_I, [_VP, _I, _PP]),
    "aq_multi_destroy": (_I, [_VP]),
    "aq_multi_shards": (_I, [_VP]),
    "aq_multi_session": (_VP, [_VP, _I]),
    "aq_multi_pq_quantize": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _I, _VP]),
    "aq_multi_adc_search": (_I, [_VP, _VP, _SZ, _SZ, _VP, _SZ, _SZ, _SZ, _VP, _SZ, _SZ, _SZ,
                                 _SZ, _VP, _VP]),
    "aq_multi_train_apq": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _SZ, _VP, _VP, _I, _VP, _VP, _VP,
                                _VP]),
    # row-sharded training building blocks
    "aq_dev_weight_flags": (_I, [_VP, _VP, _VP]),
    "aq_dev_normal_equations_partial": (_I, [_VP, _VP, _VP, _SZ, _VP, _VP, _VP, _VP]),
    "aq_dev_iso_partials": (_I, [_VP, _VP, _VP, _SZ, _VP, _VP, _VP]),
    "aq_dev_solve_normal_equations": (_I, [_VP, _VP, _VP, _SZ, C.c_double]),
    "aq_codebook_set_device": (_I, [_VP, _VP]),
    "aq_dev_point_losses": (_I, [_VP, _VP, _VP, _VP, _VP]),
    "aq_dev_sort_desc": (_I, [_VP, _VP, _VP, _SZ]),
    "aq_dev_seq_sum": (_I, [_VP, _VP, _SZ, C.c_double, _VP]),
    "aq_dev_seq_sums": (_I, [_VP, _VP, _SZ, _SZ, _SZ, _VP, _VP]),
    "aq_dev_kmeans_assign": (_I, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "aq_dev_kmeans_partials": (_I, [_VP, _VP, _SZ, _VP, _VP, _VP, _VP]),
}


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1908_10396_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None:
            continue  # declared in the header, not yet exported by this build
        fn.restype = res
        fn.argtypes = args
    return lib


def exported_symbols() -> set[str]:
    lib = C.CDLL(LIB_PATH)
    return {n for n in _SIGS if hasattr(lib, n)}
