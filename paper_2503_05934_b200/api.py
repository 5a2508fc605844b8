"""Python host API mirroring the reference's C++ interface.

Names, argument meaning and error behaviour follow
/root/reference/proj/include/netsort/{config,hybrid}.hpp:
  NetworkConfig / base_case_applies          config.hpp:20-36
  config_registry / find_config / ...        src/config.cpp:11-70
  optimized_merge_sort(a, [left, right,] cfg) hybrid.hpp:156-177
  optimized_quick_sort(a, [low, high,] cfg)   hybrid.hpp:197-216
  classical_merge_sort / classical_quick_sort hybrid.hpp:180-183, 220-223
  run_variant(variant, a)                     hybrid.hpp:225-232
Arrays are sorted IN PLACE.  ``a`` may be a CUDA tensor (device path: no
host copies, stream-ordered on torch's current stream) or a host numpy array
(the reference's call shape: copied to the GPU, sorted, copied back); keys
are int32 (the BASELINE configs) or int64 (the reference's own benchmark
type, bench.hpp:59-61), dispatched to the *_i32 / *_i64 entry points.  Everything executes in the sm_100a library through the C ABI; there
is no CPU fallback.  Configuration errors raise ValueError (the reference
throws std::invalid_argument), device errors raise NetsortError.
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import check, lib

try:  # torch is plumbing for device memory and streams
    import torch
except Exception:  # pragma: no cover - torch is present in this image
    torch = None

kMinNetworkWidth = 2
kMaxNetworkWidth = 8


class Algorithm(enum.Enum):
    merge_sort = 0
    quick_sort = 1


def algorithm_name(a: Algorithm) -> str:
    return "MergeSort" if a is Algorithm.merge_sort else "QuickSort"


@dataclass(frozen=True)
class NetworkConfig:
    name: str
    width_mask: int = 0
    varsort_max: int = 0

    def is_classic(self) -> bool:
        return self.width_mask == 0 and self.varsort_max == 0


@dataclass(frozen=True)
class SortVariant:
    algorithm: Algorithm
    config: NetworkConfig


@dataclass
class DispatchStats:
    """hybrid.hpp:18-34 (same fields and helpers)."""
    network_hits: list = field(default_factory=lambda: [0] * (kMaxNetworkWidth + 1))
    merges: int = 0
    partitions: int = 0
    max_depth: int = 0

    def total_network_hits(self) -> int:
        return sum(self.network_hits)

    def add(self, other: "DispatchStats") -> None:
        self.network_hits = [a + b for a, b in zip(self.network_hits, other.network_hits)]
        self.merges += other.merges
        self.partitions += other.partitions
        self.max_depth = max(self.max_depth, other.max_depth)


def merge_sort_dispatch_stats(n: int, cfg: "NetworkConfig") -> DispatchStats:
    """The counters the reference's merge sort records for n keys: its
    recursion shape (hybrid.hpp:81-95) depends on n and the config only.
    Quick sort's counters depend on the data's pivot splits: they come from
    the traced quick sort (quick_sort_traced)."""
    out = (C.c_uint64 * 12)()
    check(lib().ns_merge_sort_dispatch_stats(int(n), cfg.width_mask, cfg.varsort_max,
                                             C.cast(out, C.c_void_p)), "dispatch stats")
    return DispatchStats(list(out[:9]), int(out[9]), int(out[10]), int(out[11]))


def base_case_applies(size: int, cfg: NetworkConfig) -> bool:
    return bool(lib().ns_base_case_applies(int(size), cfg.width_mask, cfg.varsort_max))


def make_fixed_config(name: str, widths: Sequence[int]) -> NetworkConfig:
    mask = 0
    for w in widths:
        if w < 3 or w > kMaxNetworkWidth:
            raise ValueError(f"fixed network width must be in [3, 8], got {w}")
        mask |= 1 << w
    return NetworkConfig(name, mask, 0)


def make_varsort_config(name: str, max_width: int) -> NetworkConfig:
    if max_width < 3 or max_width > 5:
        raise ValueError(f"varsort max width must be 3, 4, or 5, got {max_width}")
    return NetworkConfig(name, 0, max_width)


def classic_config() -> NetworkConfig:
    return NetworkConfig("Classic", 0, 0)


_REGISTRY: Optional[list] = None


def config_registry() -> list:
    """The 12 presets in registry order, read from the library."""
    global _REGISTRY
    if _REGISTRY is None:
        L = lib()
        reg = []
        for i in range(L.ns_config_count()):
            name = L.ns_config_name(i).decode()
            m, v = C.c_uint32(), C.c_int()
            check(L.ns_find_config(name.encode(), C.byref(m), C.byref(v)), "ns_find_config")
            reg.append(NetworkConfig(name, m.value, v.value))
        _REGISTRY = reg
    return list(_REGISTRY)


def find_config(name: str) -> Optional[NetworkConfig]:
    for c in config_registry():
        if c.name == name:
            return c
    return None


def bundled_variants() -> list:
    return [SortVariant(a, c) for a in (Algorithm.merge_sort, Algorithm.quick_sort)
            for c in config_registry()]


def network(width: int) -> list:
    """The comparator list the kernels run for `width` (bundled_network)."""
    buf = (C.c_uint8 * 64)()
    cnt = lib().ns_network_comparators(int(width), C.cast(buf, C.c_void_p), 32)
    if cnt < 0:
        raise ValueError(f"no bundled network of width {width}")
    return [(buf[2 * i], buf[2 * i + 1]) for i in range(cnt)]


def leaf_width(cfg: NetworkConfig) -> int:
    return int(lib().ns_leaf_width(cfg.width_mask, cfg.varsort_max))


# ---- device scratch -------------------------------------------------------
# One cached scratch buffer per (device, stream): a sort's kernels only ever
# touch the scratch of the stream they run on, so sorts on different streams
# never share one, and the caching allocator's stream bookkeeping stays exact
# (the buffer is allocated while its stream is current and used only there).
# Calls that enqueue on the same stream from several host threads are
# serialised by a per-(device, stream) lock held across the enqueue, so one
# sort's kernels are all queued before the next sort's.

_SCRATCH: dict = {}
_LOCKS: dict = {}
_LOCKS_GUARD = threading.Lock()


def _key(device, stream: int):
    d = torch.device(device)
    return (d.index if d.index is not None else torch.cuda.current_device(), int(stream))


def _lock(key):
    with _LOCKS_GUARD:
        lk = _LOCKS.get(key)
        if lk is None:
            lk = _LOCKS[key] = threading.RLock()
        return lk


def scratch(nbytes: int, device, stream: Optional[int] = None) -> int:
    """Device pointer to >= nbytes of cached scratch for (device, stream)."""
    if nbytes == 0:
        return 0
    if stream is None:
        stream = torch.cuda.current_stream(torch.device(device)).cuda_stream
    key = _key(device, stream)
    buf = _SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        _SCRATCH.pop(key, None)
        buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{key[0]}")
        _SCRATCH[key] = buf
    return buf.data_ptr()


def _with_scratch(nbytes: int, t, fn):
    """fn(scratch_ptr, stream_ptr) under the (device, stream) lock."""
    strm = _stream_ptr(t)
    with _lock(_key(t.device, strm)):
        return fn(scratch(nbytes, t.device, strm), strm)


def release_scratch() -> None:
    _SCRATCH.clear()
    lib().ns_release_cache()


def _stream_ptr(t) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _is_device(a) -> bool:
    return torch is not None and isinstance(a, torch.Tensor) and a.is_cuda


def _check_tensor(a, allow_i64: bool = False):
    ok = (torch.int32, torch.int64) if allow_i64 else (torch.int32,)
    if a.dtype not in ok:
        raise ValueError(f"keys must be {' or '.join(str(t) for t in ok)}, got {a.dtype}")
    if not a.is_contiguous():
        raise ValueError("keys must be contiguous")
    return "i64" if a.dtype == torch.int64 else "i32"


def _check_host(a):
    if not isinstance(a, np.ndarray) or a.dtype not in (np.int32, np.int64) \
            or not a.flags.c_contiguous:
        raise ValueError("host keys must be a C-contiguous int32 or int64 numpy array")
    if not a.flags.writeable:
        raise ValueError("host keys must be writeable (sorted in place)")
    return "i64" if a.dtype == np.int64 else "i32"


def _range(a, left, right):
    n = len(a) if not _is_device(a) else a.numel()
    if left is None:
        left, right = 0, n - 1
    return int(left), int(right), n


def _sort(algo: int, a, left, right, cfg: NetworkConfig):
    left, right, n = _range(a, left, right)
    if right < left:  # hybrid.hpp:160, 201 — inverted range is a no-op
        return a
    if left < 0 or right >= n:
        raise ValueError("range outside the array")
    cnt = right - left + 1
    L = lib()
    what = "optimized_merge_sort" if algo == _lib.NS_MERGE_SORT else "optimized_quick_sort"
    alg = "merge" if algo == _lib.NS_MERGE_SORT else "quick"
    if _is_device(a):
        t = _check_tensor(a, allow_i64=True)
        ptr = a.data_ptr() + a.element_size() * left
        sfx = "" if t == "i32" else "_i64"
        tb = getattr(L, f"ns_{alg}_sort_temp_bytes{sfx}")(cnt)
        fn = getattr(L, f"ns_{alg}_sort_{t}")
        check(_with_scratch(tb, a, lambda tmp, strm: fn(ptr, cnt, cfg.width_mask,
                                                         cfg.varsort_max, tmp, tb, strm)), what)
    else:
        t = _check_host(a)
        ptr = a.ctypes.data + a.itemsize * left
        fn = getattr(L, f"ns_{alg}_sort_host_{t}")
        check(fn(ptr, cnt, cfg.width_mask, cfg.varsort_max), what)
    return a


def optimized_merge_sort(a, *args):
    """optimized_merge_sort(a, cfg), optimized_merge_sort(a, left, right, cfg)
    or optimized_merge_sort(a, left, right, cfg, stats) (hybrid.hpp:156-177;
    the stats form also adds the reference's DispatchStats counters)."""
    if len(args) == 1:
        return _sort(_lib.NS_MERGE_SORT, a, None, None, args[0])
    if len(args) == 4:
        left, right, cfg, stats = args
        _sort(_lib.NS_MERGE_SORT, a, left, right, cfg)
        if int(right) >= int(left):
            stats.add(merge_sort_dispatch_stats(int(right) - int(left) + 1, cfg))
        return a
    left, right, cfg = args
    return _sort(_lib.NS_MERGE_SORT, a, left, right, cfg)


def sort_host_async(src, dst, cfg: NetworkConfig, algorithm: Algorithm = Algorithm.merge_sort,
                    stream=None):
    """Stream-ordered host-array sort (ns_*_sort_host_async_i32): upload the
    int32 numpy array `src`, sort it with the config's network base case,
    download into `dst` (may be `src`), all enqueued on `stream` (a
    torch.cuda.Stream, default the current one); returns at once.  Use pinned
    host memory (e.g. torch.empty(..., pin_memory=True).numpy()) for the
    copies to overlap; synchronise the stream before reading `dst`."""
    import torch
    if _check_host(src) != "i32" or _check_host(dst) != "i32" or len(dst) != len(src):
        raise ValueError("sort_host_async: src and dst must be int32 host arrays of equal size")
    s = stream if stream is not None else torch.cuda.current_stream()
    fn = (lib().ns_merge_sort_host_async_i32 if algorithm == Algorithm.merge_sort
          else lib().ns_quick_sort_host_async_i32)
    check(fn(src.ctypes.data, dst.ctypes.data, len(src), cfg.width_mask, cfg.varsort_max,
             s.cuda_stream), "sort_host_async")
    return dst


def merge(a, left: int, mid: int, right: int):
    """merge — hybrid.hpp:186-193: stable in-place merge of the sorted runs
    a[left..mid] and a[mid+1..right] (inclusive bounds)."""
    n = a.numel() if _is_device(a) else len(a)
    left, mid, right = int(left), int(mid), int(right)
    if not (0 <= left <= mid <= right < n):
        raise ValueError("merge: need 0 <= left <= mid <= right < size")
    L = lib()
    cnt = right - left + 1
    if _is_device(a):
        t = _check_tensor(a, allow_i64=True)
        offs = (C.c_int64 * 3)(0, mid - left + 1, cnt)
        sfx = "" if t == "i32" else "_i64"
        tb = getattr(L, f"ns_merge_runs_temp_bytes{sfx}")(cnt, 2)
        fn = getattr(L, f"ns_merge_runs_{t}")
        base = a.data_ptr() + a.element_size() * left
        check(_with_scratch(tb, a, lambda tmp, strm: fn(base, C.cast(offs, C.c_void_p), 2, tmp,
                                                         tb, strm)), "merge")
    else:
        t = _check_host(a)
        check(getattr(L, f"ns_merge_host_{t}")(a.ctypes.data + a.itemsize * left,
                                               mid - left + 1, cnt), "merge")
    return a


def optimized_quick_sort(a, *args):
    """optimized_quick_sort(a, cfg), optimized_quick_sort(a, low, high, cfg)
    or optimized_quick_sort(a, low, high, cfg, stats) (hybrid.hpp:197-216).
    The stats form runs the reference's own recursion on the GPU
    (quick_sort_traced) and adds its DispatchStats counters."""
    if len(args) == 1:
        return _sort(_lib.NS_QUICK_SORT, a, None, None, args[0])
    if len(args) == 4:
        low, high, cfg, stats = args
        stats.add(quick_sort_traced(a, low, high, cfg))
        return a
    low, high, cfg = args
    return _sort(_lib.NS_QUICK_SORT, a, low, high, cfg)


def quick_sort_traced(a, low, high, cfg: NetworkConfig) -> DispatchStats:
    """Sort a[low..high] with the reference's quick sort executed node for node
    on the GPU (median_of_three + hoare_partition at every node of
    quick_sort_rec, hybrid.hpp:105-150; ns_quick_sort_traced_*) and return its
    DispatchStats.  high < low is a no-op with zero counters (hybrid.hpp:201).
    Synchronises (the instrumentation path, not the timed one)."""
    low, high, n = _range(a, low, high)
    out = (C.c_uint64 * 12)()
    if high < low:
        return DispatchStats()
    if low < 0 or high >= n:
        raise ValueError("range outside the array")
    cnt = high - low + 1
    L = lib()
    if _is_device(a):
        t = _check_tensor(a, allow_i64=True)
        ptr = a.data_ptr() + a.element_size() * low
        tb = L.ns_quick_sort_traced_temp_bytes(cnt)
        fn = getattr(L, f"ns_quick_sort_traced_{t}")
        check(_with_scratch(tb, a, lambda tmp, strm: fn(ptr, cnt, cfg.width_mask, cfg.varsort_max,
                                                         C.cast(out, C.c_void_p), tmp, tb, strm)),
              "optimized_quick_sort(stats)")
    else:
        t = _check_host(a)
        fn = getattr(L, f"ns_quick_sort_traced_host_{t}")
        check(fn(a.ctypes.data + a.itemsize * low, cnt, cfg.width_mask, cfg.varsort_max,
                 C.cast(out, C.c_void_p)), "optimized_quick_sort(stats)")
    return DispatchStats(list(out[:9]), int(out[9]), int(out[10]), int(out[11]))


def median_of_three(a, low: int, high: int) -> int:
    """median_of_three — hybrid.hpp:105-114: the three compare-exchanges on
    a[low], a[low+(high-low)//2], a[high] (in place, on the GPU) and the pivot
    a[mid]; ranges of length 1 or 2 yield a[low] untouched."""
    n = a.numel() if _is_device(a) else len(a)
    low, high = int(low), int(high)
    if not (0 <= low <= high < n):
        raise ValueError("median_of_three: need 0 <= low <= high < size")
    L = lib()
    if _is_device(a):
        t = _check_tensor(a, allow_i64=True)
        piv = (C.c_int64 if t == "i64" else C.c_int32)()
        check(getattr(L, f"ns_median_of_three_{t}")(a.data_ptr(), n, low, high, C.addressof(piv),
                                                   _stream_ptr(a)), "median_of_three")
    else:
        t = _check_host(a)
        piv = (C.c_int64 if t == "i64" else C.c_int32)()
        check(getattr(L, f"ns_median_of_three_host_{t}")(a.ctypes.data, n, low, high,
                                                        C.addressof(piv)), "median_of_three")
    return int(piv.value)


def hoare_partition(a, low: int, high: int, pivot: int) -> int:
    """hoare_partition — hybrid.hpp:121-133 on a[low..high] (low < high): the
    reference's swaps in the reference's cells, and its split j (low <= j <
    high, [low..j] <= pivot <= [j+1..high]); computed on the GPU in two
    streaming passes.  A pivot above or below every key in the range raises
    ValueError (the reference's scan would leave the range)."""
    n = a.numel() if _is_device(a) else len(a)
    low, high = int(low), int(high)
    if not (0 <= low < high < n):
        raise ValueError("hoare_partition: need 0 <= low < high < size")
    L = lib()
    split = C.c_int64()
    if _is_device(a):
        t = _check_tensor(a, allow_i64=True)
        tb = L.ns_hoare_partition_temp_bytes(high - low + 1)
        fn = getattr(L, f"ns_hoare_partition_{t}")
        check(_with_scratch(tb, a, lambda tmp, strm: fn(a.data_ptr(), n, low, high, int(pivot),
                                                         C.addressof(split), tmp, tb, strm)),
              "hoare_partition")
    else:
        t = _check_host(a)
        check(getattr(L, f"ns_hoare_partition_host_{t}")(a.ctypes.data, n, low, high, int(pivot),
                                                        C.addressof(split)), "hoare_partition")
    return int(split.value)


def classical_merge_sort(a):
    return optimized_merge_sort(a, classic_config())


def classical_quick_sort(a):
    return optimized_quick_sort(a, classic_config())


def run_variant(variant: SortVariant, a, stats: Optional[DispatchStats] = None):
    """run_variant (hybrid.hpp:225-243).  With stats, quick sort runs the
    traced reference recursion (quick_sort_traced)."""
    if stats is not None:
        n = a.numel() if _is_device(a) else len(a)
        if n == 0:  # hybrid.hpp:237
            return a
        if variant.algorithm is not Algorithm.merge_sort:
            return optimized_quick_sort(a, 0, n - 1, variant.config, stats)
        return optimized_merge_sort(a, 0, n - 1, variant.config, stats)
    if variant.algorithm is Algorithm.merge_sort:
        return optimized_merge_sort(a, variant.config)
    return optimized_quick_sort(a, variant.config)


# ---- batch entry points (BASELINE configs 2 and 4) -------------------------

def sort_small_batch(keys, offsets, status=None):
    """Sort every ragged array keys[offsets[i]:offsets[i+1]] (length <= 8) with
    its size-specific network.  keys: CUDA int32, offsets: CUDA int32/uint32
    (num_arrays + 1 entries, read as uint32).  Without `status` the call
    reads the validation result back and raises ValueError on a bad length;
    with `status` (a CUDA int32 tensor of >= 1 element) it stays stream-
    ordered (graph-capturable) and writes 0 / NS_ERR_INVALID to status[0].
    A bad length leaves every key untouched."""
    _check_tensor(keys)
    if offsets.dtype not in (torch.int32, torch.uint32) or not offsets.is_cuda:
        raise ValueError("offsets must be a CUDA int32/uint32 tensor")
    num = offsets.numel() - 1
    if status is not None:
        if status.dtype != torch.int32 or not status.is_cuda or status.numel() < 1:
            raise ValueError("status must be a CUDA int32 tensor")
        check(lib().ns_sort_small_batch_async_i32(keys.data_ptr(), offsets.data_ptr(),
                                                  max(num, 0), status.data_ptr(),
                                                  _stream_ptr(keys)), "sort_small_batch")
        return keys
    check(lib().ns_sort_small_batch_i32(keys.data_ptr(), offsets.data_ptr(), max(num, 0),
                                        _stream_ptr(keys)), "sort_small_batch")
    return keys


def segmented_sort(keys, seg_len: int, cfg: NetworkConfig,
                   algorithm: Algorithm = Algorithm.quick_sort):
    """Sort keys.numel() // seg_len back-to-back segments independently."""
    t = _check_tensor(keys, allow_i64=True)
    if seg_len <= 0 or keys.numel() % seg_len:
        raise ValueError("keys must hold a whole number of segments")
    nseg = keys.numel() // seg_len
    L = lib()
    sfx = "" if t == "i32" else "_i64"
    tb = getattr(L, f"ns_segmented_sort_temp_bytes{sfx}")(nseg, seg_len)
    fn = getattr(L, f"ns_segmented_sort_{t}")
    check(_with_scratch(tb, keys, lambda tmp, strm: fn(keys.data_ptr(), nseg, seg_len,
                                                        algorithm.value, cfg.width_mask,
                                                        cfg.varsort_max, tmp, tb, strm)),
          "segmented_sort")
    return keys


# ---- key-value --------------------------------------

def sort_pairs(keys, values=None):
    """Stable sort of CUDA int32 keys in place, carrying a 4-byte payload
    (int32/uint32/float32 CUDA tensor of the same length) through the same
    permutation: equal keys keep their input order, as the reference's
    classical merge (hybrid.hpp:61-79) keeps them."""
    _check_tensor(keys)
    n = keys.numel()
    if values is not None:
        if not values.is_cuda or values.numel() != n or values.element_size() != 4 \
                or not values.is_contiguous():
            raise ValueError("values must be a contiguous 4-byte CUDA tensor of len(keys)")
    L = lib()
    tb = L.ns_sort_pairs_temp_bytes_i32(n)
    vptr = values.data_ptr() if values is not None else None
    check(_with_scratch(tb, keys, lambda tmp, strm: L.ns_sort_pairs_i32(keys.data_ptr(), vptr, n,
                                                                         tmp, tb, strm)),
          "sort_pairs")
    return keys, values


def argsort(keys):
    """Stable argsort of CUDA int32 keys: returns an int64 tensor perm with
    keys[perm] ascending and equal keys in input order (keys unchanged)."""
    _check_tensor(keys)
    n = keys.numel()
    perm = torch.empty(n, dtype=torch.int32, device=keys.device)
    L = lib()
    tb = L.ns_argsort_temp_bytes_i32(n)
    check(_with_scratch(tb, keys, lambda tmp, strm: L.ns_argsort_i32(keys.data_ptr(),
                                                                      perm.data_ptr(), n, tmp,
                                                                      tb, strm)), "argsort")
    return perm.to(torch.int64) if n < 2**31 else perm.view(torch.uint32).to(torch.int64)


# ---- checking helpers ------------------------------------------------------

def multiset_digest(keys) -> tuple:
    """Order-independent (sum, xor) digest of mix64(key) over a CUDA tensor."""
    t = _check_tensor(keys, allow_i64=True)
    out = torch.zeros(2, dtype=torch.int64, device=keys.device)
    check(getattr(lib(), f"ns_multiset_digest_{t}")(keys.data_ptr(), keys.numel(),
                                                      out.data_ptr(), _stream_ptr(keys)),
          "multiset_digest")
    s, x = out.cpu().tolist()
    return s & (2**64 - 1), x & (2**64 - 1)


def count_inversions(keys) -> int:
    """Number of adjacent descents (0 == sorted)."""
    t = _check_tensor(keys, allow_i64=True)
    out = torch.zeros(1, dtype=torch.int64, device=keys.device)
    check(getattr(lib(), f"ns_count_inversions_{t}")(keys.data_ptr(), keys.numel(),
                                                       out.data_ptr(), _stream_ptr(keys)),
          "count_inversions")
    return int(out.item())


# ---- seeded inputs (generate, src/datagen.cpp:18-50) -------

_DIST = {"random": 0, "sorted": 1, "nearly_sorted": 2}


def generate(dist: str, n: int, seed: int = 42, p: float = 0.01, dtype=np.int32) -> np.ndarray:
    """Host array of the reference's distributions: random (int32: next() >> 33,
    int64: next()), sorted 0..n-1, nearly_sorted (ramp + floor(p*n) swaps)."""
    if dist not in _DIST:
        raise ValueError(f"unknown distribution {dist!r}")
    a = np.empty(int(n), dtype=dtype)
    sfx = "i64" if a.dtype == np.int64 else "i32"
    check(getattr(lib(), f"ns_generate_host_{sfx}")(a.ctypes.data, a.size, _DIST[dist],
                                                     int(seed) % 2**64, float(p)), "generate")
    return a


def generate_batch(num_arrays: int, seed: int = 42):
    """(offsets uint32[num_arrays + 1], keys int32[K]) of the ragged base-case
    batch (lengths U{3..8})."""
    L = lib()
    k = L.ns_generate_batch_host_i32(int(num_arrays), int(seed) % 2**64, None, None)
    offs = np.empty(int(num_arrays) + 1, dtype=np.uint32)
    keys = np.empty(int(k), dtype=np.int32)
    L.ns_generate_batch_host_i32(int(num_arrays), int(seed) % 2**64, offs.ctypes.data,
                                 keys.ctypes.data)
    return offs, keys
