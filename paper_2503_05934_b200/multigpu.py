"""Multi-GPU host layer behind ONE host thread.

Python face of the C ABI's single-process multi-device entry points
(include/netsort_b200.h, "multi-GPU, one host thread"):

  sample_sort_multi(shards, exchange)   BASELINE config 5: one array sharded
                                        over devices, PSRS sample sort, device
                                        d returns the d-th key range
  shard_batch_plan(offsets, nshards)    array ranges of ~equal key counts
  sort_small_batch_multi(...)           configs 2 / 4 sharded by array
  segmented_sort_multi(...)

The one-process-per-GPU form over torch.distributed is samplesort.py; both
share the per-device steps of the library.  NCCL (exchange="nccl") is loaded
by the library at run time; exchange="p2p" merges straight out of the peers'
memory and also accepts several shards on one device (virtual ranks).
"""
from __future__ import annotations

import ctypes as C
from typing import List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import check, lib

_EXCHANGE = {"nccl": _lib.NS_EXCHANGE_NCCL, "p2p": _lib.NS_EXCHANGE_P2P}


def _arr(ctype, vals):
    return (ctype * len(vals))(*vals)


def nccl_available() -> bool:
    return bool(lib().ns_nccl_available())


class NcclComms:
    """Single-process communicators over `devices` (ncclCommInitAll)."""

    def __init__(self, devices: Sequence[int]):
        self.devices = list(devices)
        self.handle = (C.c_void_p * len(self.devices))()
        check(lib().ns_nccl_comms_init_all(len(self.devices), _arr(C.c_int, self.devices),
                                           self.handle), "ncclCommInitAll")

    def close(self):
        if self.handle is not None:
            check(lib().ns_nccl_comms_destroy(len(self.devices), self.handle), "ncclCommDestroy")
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def sample_sort_plan(bounds: np.ndarray):
    """(recv_offsets [g, g+1], recv_totals [g]) from the g x (g+1) bucket
    bounds of the sorted shards (host logic of the exchange)."""
    b = np.ascontiguousarray(bounds, dtype=np.int64)
    g = b.shape[0]
    ro = np.empty((g, g + 1), np.int64)
    rt = np.empty(g, np.int64)
    check(lib().ns_sample_sort_plan(g, b.ctypes.data, ro.ctypes.data, rt.ctypes.data),
          "sample_sort_plan")
    return ro, rt


def sample_sort_multi(shards: List[torch.Tensor], cfg=None, exchange: str = "p2p",
                      comms: Optional[NcclComms] = None, out_capacity: Optional[int] = None
                      ) -> List[torch.Tensor]:
    """Globally sort the array whose pieces are `shards` (CUDA int32 tensors,
    one per device, possibly several on one device for exchange="p2p").
    Returns one tensor per shard: shard d's output holds the d-th key range;
    concatenated in order they are the sorted array.  Shards are sorted in
    place as a side effect."""
    from .api import find_config
    cfg = cfg or find_config("6To8")
    g = len(shards)
    devs = [t.device.index for t in shards]
    for t in shards:
        if t.dtype != torch.int32 or not t.is_cuda or not t.is_contiguous():
            raise ValueError("shards must be contiguous CUDA int32 tensors")
    if exchange not in _EXCHANGE:
        raise ValueError("exchange must be 'nccl' or 'p2p'")
    if exchange == "nccl" and comms is None:
        raise ValueError("exchange='nccl' needs NcclComms")
    total = sum(t.numel() for t in shards)
    cap = out_capacity or max(1, min(total, 2 * max(t.numel() for t in shards) + 4096 * g))
    L = lib()
    shard_max = max(t.numel() for t in shards)
    tb = L.ns_sample_sort_multi_temp_bytes(g, shard_max, cap)
    while True:
        outs = [torch.empty(cap, dtype=torch.int32, device=t.device) for t in shards]
        temps = [torch.empty(tb, dtype=torch.uint8, device=t.device) for t in shards]
        streams = [torch.cuda.current_stream(t.device).cuda_stream for t in shards]
        counts = (C.c_size_t * g)(*[t.numel() for t in shards])
        oc = (C.c_size_t * g)()
        st = L.ns_sample_sort_multi_i32(
            g, _arr(C.c_int, devs), comms.handle if comms is not None else None,
            _EXCHANGE[exchange], _arr(C.c_void_p, [t.data_ptr() for t in shards]), counts,
            _arr(C.c_void_p, [o.data_ptr() for o in outs]), cap, oc, cfg.width_mask,
            cfg.varsort_max, _arr(C.c_void_p, [t.data_ptr() for t in temps]), tb,
            _arr(C.c_void_p, streams))
        if st == _lib.NS_ERR_TEMP and max(oc) > cap:  # a bucket above the PSRS estimate
            cap = int(max(oc))
            tb = L.ns_sample_sort_multi_temp_bytes(g, shard_max, cap)
            continue
        check(st, "sample_sort_multi")
        return [o[: int(oc[d])] for d, o in enumerate(outs)]


def shard_batch_plan(offsets: np.ndarray, nshards: int) -> np.ndarray:
    """Array index bounds [nshards + 1] of a key-balanced split of a ragged
    batch (offsets: num_arrays + 1 uint32)."""
    o = np.ascontiguousarray(offsets, dtype=np.uint32)
    out = np.empty(nshards + 1, dtype=np.uint64)
    check(lib().ns_shard_batch_plan(o.ctypes.data, max(o.size - 1, 0), nshards, out.ctypes.data),
          "shard_batch_plan")
    return out.astype(np.int64)


def shard_batch(offsets: np.ndarray, keys: np.ndarray, nshards: int):
    """[(rebased offsets, keys)] per shard of a ragged batch."""
    ab = shard_batch_plan(offsets, nshards)
    out = []
    for k in range(nshards):
        a0, a1 = int(ab[k]), int(ab[k + 1])
        k0, k1 = int(offsets[a0]), int(offsets[a1])
        out.append(((offsets[a0:a1 + 1] - offsets[a0]).astype(np.uint32), keys[k0:k1]))
    return out


def sort_small_batch_multi(keys: List[torch.Tensor], offsets: List[torch.Tensor]) -> List[int]:
    """Each device sorts its own shard of a ragged batch (no collective);
    returns the per-device status (0 ok, NS_ERR_INVALID)."""
    g = len(keys)
    status = [torch.ones(1, dtype=torch.int32, device=k.device) for k in keys]
    check(lib().ns_sort_small_batch_multi_i32(
        g, _arr(C.c_int, [k.device.index for k in keys]),
        _arr(C.c_void_p, [k.data_ptr() for k in keys]),
        _arr(C.c_void_p, [o.data_ptr() for o in offsets]),
        (C.c_size_t * g)(*[max(o.numel() - 1, 0) for o in offsets]),
        _arr(C.c_void_p, [s.data_ptr() for s in status]),
        _arr(C.c_void_p, [torch.cuda.current_stream(k.device).cuda_stream for k in keys])),
        "sort_small_batch_multi")
    return [int(s.item()) for s in status]


def segmented_sort_multi(keys: List[torch.Tensor], seg_len: int, cfg=None,
                         algorithm=None) -> None:
    """Each device sorts its own whole segments (no collective)."""
    from .api import Algorithm, find_config
    cfg = cfg or find_config("3To5")
    algorithm = algorithm or Algorithm.quick_sort
    g = len(keys)
    L = lib()
    nseg = [k.numel() // seg_len for k in keys]
    if any(k.numel() % seg_len for k in keys):
        raise ValueError("every shard must hold whole segments")
    tbs = [L.ns_segmented_sort_temp_bytes(s, seg_len) for s in nseg]
    temps = [torch.empty(max(tb, 1), dtype=torch.uint8, device=k.device) for k, tb in zip(keys, tbs)]
    check(L.ns_segmented_sort_multi_i32(
        g, _arr(C.c_int, [k.device.index for k in keys]),
        _arr(C.c_void_p, [k.data_ptr() for k in keys]), (C.c_size_t * g)(*nseg), seg_len,
        algorithm.value, cfg.width_mask, cfg.varsort_max,
        _arr(C.c_void_p, [t.data_ptr() for t in temps]), (C.c_size_t * g)(*tbs),
        _arr(C.c_void_p, [torch.cuda.current_stream(k.device).cuda_stream for k in keys])),
        "segmented_sort_multi")
