"""ctypes front-end to the CPU oracle (oracle/_build/liboracle.so) and to the
reference itself (oracle/_ref/libnetsort_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() (as the
checker) and bench.py's cpu_baseline / --impl reference legs.  The product
package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnetsort_ref.so")

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")

KIND = {"random": 0, "sorted": 1, "nearly_sorted": 2}

# Restates config_registry — /root/reference/proj/src/config.cpp:35-53.
# (name, width_mask, varsort_max); the product's own table lives in the C++
# host layer and is pinned against this one and against oracle/_ref.
REGISTRY = [
    ("Classic", 0, 0),
    ("PowerOf2", (1 << 4) | (1 << 8), 0),
    ("Even", (1 << 4) | (1 << 6) | (1 << 8), 0),
    ("Odd", (1 << 3) | (1 << 5) | (1 << 7), 0),
    ("3", 1 << 3, 0),
    ("3To4", (1 << 3) | (1 << 4), 0),
    ("3To5", (1 << 3) | (1 << 4) | (1 << 5), 0),
    ("3To8", sum(1 << w for w in range(3, 9)), 0),
    ("6To8", (1 << 6) | (1 << 7) | (1 << 8), 0),
    ("VarSort3", 0, 3),
    ("VarSort4", 0, 4),
    ("VarSort5", 0, 5),
]
CONFIGS = {n: (m, v) for n, m, v in REGISTRY}


class OracleStats(C.Structure):
    _fields_ = [("network_hits", C.c_uint64 * 9), ("merges", C.c_uint64),
                ("partitions", C.c_uint64), ("max_depth", C.c_int32)]


def build(harness: bool = False) -> None:
    """Build the oracle (and oracle/_ref when /root/reference is present);
    harness=True also links the reference's benchmark harness against the
    product library (oracle/_ref/harness_gpu, needs the library built)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"] + (["harness"] if harness else []),
                   check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.oracle_splitmix64_next.argtypes = [C.POINTER(C.c_uint64)]
        L.oracle_splitmix64_next.restype = C.c_uint64
        L.oracle_generate_i32.argtypes = [C.c_int, C.c_size_t, C.c_uint64, C.c_double, _i32p]
        L.oracle_generate_i64.argtypes = [C.c_int, C.c_size_t, C.c_uint64, C.c_double, _i64p]
        L.oracle_generate_batch_i32.argtypes = [C.c_size_t, C.c_uint64, C.c_void_p, C.c_void_p]
        L.oracle_generate_batch_i32.restype = C.c_size_t
        L.oracle_network.argtypes = [C.c_int, _u8p, C.c_int]
        L.oracle_sort_small_i32.argtypes = [_i32p, C.c_int]
        L.oracle_base_case_applies.argtypes = [C.c_int64, C.c_uint32, C.c_int]
        L.oracle_merge_sort_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                            C.c_void_p]
        L.oracle_merge_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_median_of_three_i32.argtypes = [_i32p, C.c_int64, C.c_int64]
        L.oracle_median_of_three_i32.restype = C.c_int32
        L.oracle_hoare_partition_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int32]
        L.oracle_hoare_partition_i32.restype = C.c_int64
        L.oracle_quick_sort_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                            C.c_void_p]
        L.oracle_sort_small_batch_i32.argtypes = [_i32p, _u32p, C.c_size_t]
        L.oracle_segmented_quick_sort_i32.argtypes = [_i32p, C.c_size_t, C.c_size_t,
                                                      C.c_uint32, C.c_int]
        L.oracle_multiset_digest_i32.argtypes = [_i32p, C.c_size_t, _u64p]
        L.oracle_stable_sort_pairs_i32.argtypes = [_i32p, _u32p, C.c_int64]
        # int64 instantiations (netsort_oracle_sort.inc with KEY = int64_t)
        L.oracle_sort_small_i64.argtypes = [_i64p, C.c_int]
        L.oracle_merge_sort_i64.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                            C.c_void_p]
        L.oracle_merge_i64.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_median_of_three_i64.argtypes = [_i64p, C.c_int64, C.c_int64]
        L.oracle_median_of_three_i64.restype = C.c_int64
        L.oracle_hoare_partition_i64.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_int64]
        L.oracle_hoare_partition_i64.restype = C.c_int64
        L.oracle_quick_sort_i64.argtypes = [_i64p, C.c_int64, C.c_int64, C.c_uint32, C.c_int,
                                            C.c_void_p]
        L.oracle_multiset_digest_i64.argtypes = [_i64p, C.c_size_t, _u64p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference compiled from /root/reference (oracle/_ref)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        R = C.CDLL(REF_SO)
        R.ref_find_config.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_int)]
        R.ref_config_count.restype = C.c_int
        R.ref_config_name.argtypes = [C.c_int]
        R.ref_config_name.restype = C.c_char_p
        R.ref_merge_sort_i32.argtypes = [_i32p, C.c_int64, C.c_uint32, C.c_int, C.c_void_p]
        R.ref_quick_sort_i32.argtypes = [_i32p, C.c_int64, C.c_uint32, C.c_int, C.c_void_p]
        R.ref_merge_sort_range_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int64,
                                               C.c_uint32, C.c_int]
        R.ref_quick_sort_range_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int64,
                                               C.c_uint32, C.c_int]
        R.ref_sort_small_i32.argtypes = [_i32p, C.c_int]
        R.ref_sort_small_batch_i32.argtypes = [_i32p, _u32p, C.c_int64]
        R.ref_segmented_quick_sort_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_uint32,
                                                   C.c_int]
        R.ref_network.argtypes = [C.c_int, _u8p, C.c_int]
        R.ref_median_of_three_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int64]
        R.ref_median_of_three_i32.restype = C.c_int32
        R.ref_hoare_partition_i32.argtypes = [_i32p, C.c_int64, C.c_int64, C.c_int64, C.c_int32]
        R.ref_hoare_partition_i32.restype = C.c_int64
        R.ref_merge_sort_i64.argtypes = [_i64p, C.c_int64, C.c_uint32, C.c_int, C.c_void_p]
        R.ref_quick_sort_i64.argtypes = [_i64p, C.c_int64, C.c_uint32, C.c_int, C.c_void_p]
        R.ref_generate_i64.argtypes = [C.c_int, C.c_int64, C.c_uint64, C.c_double, _i64p]
        R.ref_splitmix64_nth.argtypes = [C.c_uint64, C.c_int64]
        R.ref_splitmix64_nth.restype = C.c_uint64
        _ref = R
    return _ref


# ---- convenience wrappers (numpy in, numpy out) ---------------------------

def generate_i32(kind: str, n: int, seed: int = 42, p: float = 0.01) -> np.ndarray:
    out = np.empty(n, np.int32)
    rc = lib().oracle_generate_i32(KIND[kind], n, seed, p, out)
    if rc != 0:
        raise ValueError("perturbation must lie in [0, 1]")
    return out


def generate_i64(kind: str, n: int, seed: int = 42, p: float = 0.01) -> np.ndarray:
    out = np.empty(n, np.int64)
    rc = lib().oracle_generate_i64(KIND[kind], n, seed, p, out)
    if rc != 0:
        raise ValueError("perturbation must lie in [0, 1]")
    return out


def generate_batch_i32(num_arrays: int, seed: int = 42):
    total = lib().oracle_generate_batch_i32(num_arrays, seed, None, None)
    offsets = np.empty(num_arrays + 1, np.uint32)
    keys = np.empty(total, np.int32)
    lib().oracle_generate_batch_i32(num_arrays, seed, offsets.ctypes.data, keys.ctypes.data)
    return offsets, keys


def network(width: int):
    buf = np.zeros(64, np.uint8)
    cnt = lib().oracle_network(width, buf, 32)
    if cnt < 0:
        raise ValueError(f"no bundled network of width {width}")
    return [(int(buf[2 * i]), int(buf[2 * i + 1])) for i in range(cnt)]


def _keys(a: np.ndarray):
    """int64 arrays keep their type (the *_i64 instantiation); anything else
    is taken as int32 (the BASELINE configs)."""
    if isinstance(a, np.ndarray) and a.dtype == np.int64:
        return np.ascontiguousarray(a).copy(), "i64"
    return np.ascontiguousarray(a, np.int32).copy(), "i32"


def merge_sort(a: np.ndarray, config: str = "6To8", stats: bool = False):
    mask, vs = CONFIGS[config]
    a, t = _keys(a)
    st = OracleStats()
    getattr(lib(), f"oracle_merge_sort_{t}")(a, 0, len(a) - 1, mask, vs,
                                             C.addressof(st) if stats else None)
    return (a, st) if stats else a


def quick_sort(a: np.ndarray, config: str = "3To5", stats: bool = False):
    mask, vs = CONFIGS[config]
    a, t = _keys(a)
    st = OracleStats()
    getattr(lib(), f"oracle_quick_sort_{t}")(a, 0, len(a) - 1, mask, vs,
                                             C.addressof(st) if stats else None)
    return (a, st) if stats else a


def sort_small_batch(keys: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    k = np.ascontiguousarray(keys, np.int32).copy()
    lib().oracle_sort_small_batch_i32(k, np.ascontiguousarray(offsets, np.uint32),
                                      len(offsets) - 1)
    return k


def segmented_quick_sort(keys: np.ndarray, seg_len: int, config: str = "3To5") -> np.ndarray:
    mask, vs = CONFIGS[config]
    k = np.ascontiguousarray(keys, np.int32).copy()
    lib().oracle_segmented_quick_sort_i32(k, len(k) // seg_len, seg_len, mask, vs)
    return k


def multiset_digest(a: np.ndarray):
    out = np.zeros(2, np.uint64)
    a, t = _keys(a)
    getattr(lib(), f"oracle_multiset_digest_{t}")(a, len(a), out)
    return int(out[0]), int(out[1])


def stable_sort_pairs(keys: np.ndarray, values: np.ndarray):
    """Classical stable merge sort of (key, payload) pairs (hybrid.hpp:61-95)."""
    k = np.ascontiguousarray(keys, np.int32).copy()
    v = np.ascontiguousarray(values, np.uint32).copy()
    lib().oracle_stable_sort_pairs_i32(k, v, len(k))
    return k, v
