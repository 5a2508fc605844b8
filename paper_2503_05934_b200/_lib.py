"""ctypes binding of the C ABI (include/netsort_b200.h).

This is the Python-side equivalent of the binding a reference maintainer
would add: every symbol the header declares is declared here
with its exact argument types.  The library is built in-tree by
``paper_2503_05934_b200/csrc/Makefile``; there is no fallback — if it is
missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
# NETSORT_B200_LIB: an alternative build of the same library (A/B runs of a
# compile-time variant, tools/build_variant.sh); the ABI is identical
LIB_PATH = os.environ.get("NETSORT_B200_LIB") or os.path.join(PKG, "lib", "libnetsort_b200.so")
CSRC = os.path.join(PKG, "csrc")

NS_OK, NS_ERR_INVALID, NS_ERR_CUDA, NS_ERR_OOM, NS_ERR_TEMP, NS_ERR_NCCL = 0, 1, 2, 3, 4, 5
NS_EXCHANGE_NCCL, NS_EXCHANGE_P2P = 0, 1
NS_MERGE_SORT, NS_QUICK_SORT = 0, 1

_vp, _sz, _u32, _i32, _i64 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_int, C.c_int64

# name -> (restype, argtypes); the complete C ABI.
SIGNATURES = {
    "ns_status_string": (C.c_char_p, [_i32]),
    "ns_last_error": (C.c_char_p, []),
    "ns_version": (_i32, []),
    "ns_find_config": (_i32, [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int)]),
    "ns_config_count": (_i32, []),
    "ns_config_name": (C.c_char_p, [_i32]),
    "ns_base_case_applies": (_i32, [_i64, _u32, _i32]),
    "ns_leaf_width": (_i32, [_u32, _i32]),
    "ns_network_comparators": (_i32, [_i32, _vp, _i32]),
    "ns_merge_sort_dispatch_stats": (_i32, [_i64, _u32, _i32, _vp]),
    "ns_merge_sort_temp_bytes": (_sz, [_sz]),
    "ns_merge_sort_i32": (_i32, [_vp, _sz, _u32, _i32, _vp, _sz, _vp]),
    "ns_merge_sort_temp_bytes_i64": (_sz, [_sz]),
    "ns_merge_sort_i64": (_i32, [_vp, _sz, _u32, _i32, _vp, _sz, _vp]),
    "ns_quick_sort_temp_bytes": (_sz, [_sz]),
    "ns_quick_sort_temp_bytes_i64": (_sz, [_sz]),
    "ns_quick_sort_i64": (_i32, [_vp, _sz, _u32, _i32, _vp, _sz, _vp]),
    "ns_quick_sort_i32": (_i32, [_vp, _sz, _u32, _i32, _vp, _sz, _vp]),
    "ns_sort_small_batch_i32": (_i32, [_vp, _vp, _sz, _vp]),
    "ns_merge_sort_host_async_i32": (_i32, [_vp, _vp, _sz, _u32, _i32, _vp]),
    "ns_quick_sort_host_async_i32": (_i32, [_vp, _vp, _sz, _u32, _i32, _vp]),
    "ns_sort_small_batch_async_i32": (_i32, [_vp, _vp, _sz, _vp, _vp]),
    "ns_sort_pairs_temp_bytes_i32": (_sz, [_sz]),
    "ns_sort_pairs_i32": (_i32, [_vp, _vp, _sz, _vp, _sz, _vp]),
    "ns_argsort_temp_bytes_i32": (_sz, [_sz]),
    "ns_argsort_i32": (_i32, [_vp, _vp, _sz, _vp, _sz, _vp]),
    "ns_segmented_sort_temp_bytes": (_sz, [_sz, _sz]),
    "ns_segmented_sort_i32": (_i32, [_vp, _sz, _sz, _i32, _u32, _i32, _vp, _sz, _vp]),
    "ns_segmented_sort_temp_bytes_i64": (_sz, [_sz, _sz]),
    "ns_segmented_sort_i64": (_i32, [_vp, _sz, _sz, _i32, _u32, _i32, _vp, _sz, _vp]),
    "ns_regular_samples_i32": (_i32, [_vp, _sz, _i32, _vp, _vp]),
    "ns_select_splitters_i32": (_i32, [_vp, _i32, _i32, _vp, _vp]),
    "ns_bucket_bounds_i32": (_i32, [_vp, _sz, _vp, _i32, _vp, _vp]),
    "ns_merge_runs_temp_bytes": (_sz, [_sz, _i32]),
    "ns_merge_runs_i32": (_i32, [_vp, _vp, _i32, _vp, _sz, _vp]),
    "ns_merge_runs_temp_bytes_i64": (_sz, [_sz, _i32]),
    "ns_merge_runs_i64": (_i32, [_vp, _vp, _i32, _vp, _sz, _vp]),
    "ns_merge_pairs_temp_bytes": (_sz, [_i64, _i32]),
    "ns_merge_pairs_i32": (_i32, [_vp, _vp, _vp, _vp, _i32, _vp, _vp, _sz, _vp]),
    "ns_nccl_available": (_i32, []),
    "ns_nccl_comms_init_all": (_i32, [_i32, _vp, _vp]),
    "ns_nccl_comms_destroy": (_i32, [_i32, _vp]),
    "ns_sample_sort_plan": (_i32, [_i32, _vp, _vp, _vp]),
    "ns_sample_sort_multi_temp_bytes": (_sz, [_i32, _sz, _sz]),
    "ns_sample_sort_multi_i32": (_i32, [_i32, _vp, _vp, _i32, _vp, _vp, _vp, _sz, _vp, _u32, _i32,
                                        _vp, _sz, _vp]),
    "ns_shard_batch_plan": (_i32, [_vp, _sz, _i32, _vp]),
    "ns_sort_small_batch_multi_i32": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "ns_segmented_sort_multi_i32": (_i32, [_i32, _vp, _vp, _vp, _sz, _i32, _u32, _i32, _vp, _vp,
                                           _vp]),
    "ns_ipc_get_handle": (_i32, [_vp, _vp, C.POINTER(C.c_uint64)]),
    "ns_ipc_open_handle": (_i32, [_vp, C.POINTER(C.c_void_p)]),
    "ns_ipc_close": (_i32, [_vp]),
    "ns_multiset_digest_i32": (_i32, [_vp, _sz, _vp, _vp]),
    "ns_count_inversions_i32": (_i32, [_vp, _sz, _vp, _vp]),
    "ns_multiset_digest_i64": (_i32, [_vp, _sz, _vp, _vp]),
    "ns_count_inversions_i64": (_i32, [_vp, _sz, _vp, _vp]),
    "ns_generate_i32": (_i32, [_vp, _sz, _i32, C.c_uint64, _vp]),
    "ns_generate_host_i32": (_i32, [_vp, _sz, _i32, C.c_uint64, C.c_double]),
    "ns_generate_host_i64": (_i32, [_vp, _sz, _i32, C.c_uint64, C.c_double]),
    "ns_generate_batch_host_i32": (_sz, [_sz, C.c_uint64, _vp, _vp]),
    "ns_launch_count": (C.c_uint64, []),
    "ns_profile_enable": (_i32, [_i32]),
    "ns_profile_kinds": (_i32, []),
    "ns_profile_kind_name": (C.c_char_p, [_i32]),
    "ns_profile_read": (_i32, [_i32, C.POINTER(C.c_double), C.POINTER(C.c_uint64)]),
    "ns_merge_sort_host_i32": (_i32, [_vp, _sz, _u32, _i32]),
    "ns_merge_sort_host_i64": (_i32, [_vp, _sz, _u32, _i32]),
    "ns_merge_host_i32": (_i32, [_vp, _sz, _sz]),
    "ns_merge_host_i64": (_i32, [_vp, _sz, _sz]),
    "ns_quick_sort_host_i64": (_i32, [_vp, _sz, _u32, _i32]),
    "ns_quick_sort_host_i32": (_i32, [_vp, _sz, _u32, _i32]),
    "ns_release_cache": (_i32, []),
    "ns_quick_sort_traced_temp_bytes": (_sz, [_sz]),
    "ns_quick_sort_traced_i32": (_i32, [_vp, _sz, _u32, _i32, _vp, _vp, _sz, _vp]),
    "ns_quick_sort_traced_i64": (_i32, [_vp, _sz, _u32, _i32, _vp, _vp, _sz, _vp]),
    "ns_hoare_partition_temp_bytes": (_sz, [_sz]),
    "ns_hoare_partition_i32": (_i32, [_vp, _sz, _i64, _i64, C.c_int32, _vp, _vp, _sz, _vp]),
    "ns_hoare_partition_i64": (_i32, [_vp, _sz, _i64, _i64, C.c_int64, _vp, _vp, _sz, _vp]),
    "ns_median_of_three_i32": (_i32, [_vp, _sz, _i64, _i64, _vp, _vp]),
    "ns_median_of_three_i64": (_i32, [_vp, _sz, _i64, _i64, _vp, _vp]),
    "ns_quick_sort_traced_host_i32": (_i32, [_vp, _sz, _u32, _i32, _vp]),
    "ns_quick_sort_traced_host_i64": (_i32, [_vp, _sz, _u32, _i32, _vp]),
    "ns_hoare_partition_host_i32": (_i32, [_vp, _sz, _i64, _i64, C.c_int32, _vp]),
    "ns_hoare_partition_host_i64": (_i32, [_vp, _sz, _i64, _i64, C.c_int64, _vp]),
    "ns_median_of_three_host_i32": (_i32, [_vp, _sz, _i64, _i64, _vp]),
    "ns_median_of_three_host_i64": (_i32, [_vp, _sz, _i64, _i64, _vp]),
}


class NetsortError(RuntimeError):
    def __init__(self, status: int, what: str):
        lib = _LIB
        msg = lib.ns_status_string(status).decode() if lib else str(status)
        detail = lib.ns_last_error().decode() if lib else ""
        super().__init__(f"{what}: {msg}" + (f" ({detail})" if detail else ""))
        self.status = status


_LIB = None


CHECKED_LIB_PATH = os.path.join(PKG, "lib", "libnetsort_b200_checked.so")


def build(verbose: bool = False, checked: bool = True) -> str:
    """Compile the sm_100a library in-tree (nvcc cross-compiles without a GPU)
    and, with `checked`, its bounds-checked twin (NSB_CHECKED=1, used only by
    tests/test_checked_build.py)."""
    targets = ["all", "checked"] if checked else ["all"]
    subprocess.run(["make", "-s", "-C", CSRC, f"-j{os.cpu_count() or 4}"] + targets, check=True,
                   stdout=None if verbose else subprocess.DEVNULL)
    return LIB_PATH


def lib():
    """Load the C-ABI library; raises if it is absent (no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"{LIB_PATH} is missing: run `make -C {CSRC}` (or __graft_entry__.build())")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = L
    return _LIB


def check(status: int, what: str) -> None:
    if status != NS_OK:
        if status == NS_ERR_INVALID:
            raise ValueError(NetsortError(status, what).args[0])
        raise NetsortError(status, what)
