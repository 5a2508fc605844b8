#!/usr/bin/env python
"""CPU arm of bench.py: the REFERENCE's own sorts (oracle/_ref, compiled
from /root/reference/proj by oracle/Makefile) timed on ONE pinned host core.

TEST / MEASUREMENT INFRASTRUCTURE ONLY (bench.py's cpu_baseline leg and its
--impl reference arm); the product never imports it.  It runs in its own
child process so that CLOCK_PROCESS_CPUTIME_ID sees nothing but the sort:
the process pins itself to one core, loads numpy and the reference .so only,
and times each BASELINE cell with the reference harness's policy restated at
int32 (ref_measure_i32 in oracle/ref_shim.cpp, after measure_loop,
/root/reference/proj/src/bench.cpp:39-89): one untimed warm-up, untimed
refill before every call, CPU time per call, batches doubling until the CPU
total reaches --min-ms (the reference's campaign default is 500 ms,
bench.hpp:75-80).  Cells whose single call exceeds that get one timed call.

  python oracle/cpu_ref_bench.py --cells all            # every BASELINE cell
  python oracle/cpu_ref_bench.py --steps K --warmup W   # --impl reference arm

Prints one JSON object on stdout.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import platform
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

SEED = 42
OPS = {"merge": 0, "quick": 1, "batch": 2, "segmented": 3}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or None


def pin_one_core():
    cores = sorted(os.sched_getaffinity(0))
    core = cores[0]
    os.sched_setaffinity(0, {core})
    return core, len(cores), os.cpu_count()


def _ref():
    R = O.ref()
    if not hasattr(R, "_measure_bound"):
        R.ref_measure_i32.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                      C.c_int64, C.c_uint32, C.c_int, C.c_int64, C.c_void_p]
        R.ref_time_once_i32.argtypes = [C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                        C.c_int64, C.c_uint32, C.c_int, C.c_void_p]
        R._measure_bound = True
    return R


def measure(op, keys, cfg="6To8", offsets=None, count=0, seg_len=0, min_ms=500.0):
    """One cell under the reference policy; returns per-call CPU ms etc."""
    mask, vs = O.CONFIGS[cfg]
    out = (C.c_double * 4)()
    st = _ref().ref_measure_i32(OPS[op], keys.ctypes.data, keys.size,
                                offsets.ctypes.data if offsets is not None else None, count,
                                seg_len, mask, vs, int(min_ms * 1e6), C.cast(out, C.c_void_p))
    if st != 0:
        raise RuntimeError("ref_measure_i32 failed")
    it, cpu, wall, cap = out[0], out[1], out[2], out[3]
    return {"cpu_ms": cpu / it / 1e6, "wall_ms": wall / it / 1e6, "iterations": int(it),
            "cap_hit": bool(cap)}


def cell_inputs(name):
    """(op, cfg, keys, offsets, count, seg_len, keys_per_call, note) of one cell."""
    algo, cfg, dist, n = name.split(":")
    n = int(n)
    if algo == "batch":
        offs, keys = O.generate_batch_i32(n, SEED)
        return "batch", "6To8", keys, offs, n, 0, keys.size, f"{n} ragged arrays, {keys.size} keys"
    if algo == "segmented":
        nseg, seg_len = (int(x) for x in dist.split("x"))
        sample = min(nseg, n)  # n = segments actually timed
        keys = O.generate_i32("random", sample * seg_len, SEED)
        return ("segmented", cfg, keys, None, sample, seg_len, sample * seg_len,
                f"{sample} of {nseg} segments of {seg_len} keys timed; per-key rate "
                f"extrapolated to the full batch")
    keys = O.generate_i32(dist, n, SEED)
    return algo, cfg, keys, None, 0, 0, n, ""


# Every BASELINE cell (configs[0..4]); segmented: 1,024 of the 65,536 x
# 16,384 segments; C5's 2^30 merge sort: a 2^24-key sample.
CELLS = (["merge:6To8:random:10000"] +
         [f"merge:6To8:{d}:{n}" for n in (25_000, 100_000, 1_000_000)
          for d in ("random", "sorted", "nearly_sorted")] +
         [f"quick:3To5:{d}:{n}" for n in (10_000, 1_000_000, 16_777_216)
          for d in ("sorted", "random")] +
         ["segmented:3To5:65536x16384:1024", "batch:6To8:random:16777216",
          "merge:6To8:random:16777216"])


def run_cells(cells, min_ms):
    out = {}
    for c in cells:
        op, cfg, keys, offs, count, seg_len, kpc, note = cell_inputs(c)
        r = measure(op, keys, cfg, offs, count, seg_len, min_ms)
        r["keys_per_call"] = int(kpc)
        r["gkeys_per_s"] = kpc / (r["cpu_ms"] * 1e-3) / 1e9
        if note:
            r["note"] = note
        out[c] = r
    return out


def run_steps(steps, warmup, n, threads_all):
    """--impl reference: each step = one optimized_merge_sort<int32_t>(6To8) of
    an n-key uniform-random sample of the bench workload on the pinned core,
    CPU time per call (refill untimed).  Then a separate all-cores figure:
    every allowed core sorts its own independent array (not the reference's
    single-threaded path)."""
    mask, vs = O.CONFIGS["6To8"]
    src = O.generate_i32("random", n, SEED)
    work = src.copy()
    R = _ref()
    out = (C.c_double * 2)()
    cpu, wall = [], []
    for i in range(warmup + steps):
        np.copyto(work, src)
        R.ref_time_once_i32(0, work.ctypes.data, n, None, 0, 0, mask, vs, C.cast(out, C.c_void_p))
        if i >= warmup:
            cpu.append(out[0])
            wall.append(out[1])
    assert np.all(work[:-1] <= work[1:])
    res = {"cpu_ms_per_step": sum(cpu) / len(cpu) / 1e6,
           "wall_ms_per_step": sum(wall) / len(wall) / 1e6, "keys_per_step": n}
    # all cores (threads release the GIL inside the ctypes call)
    os.sched_setaffinity(0, threads_all)
    m = 1 << 22
    arrs = [O.generate_i32("random", m, SEED + t) for t in range(len(threads_all))]
    ws = [a.copy() for a in arrs]

    def one(w):
        O.ref().ref_merge_sort_i32(w, w.size, mask, vs, None)

    dts = []
    for rep in range(3):
        for w, a in zip(ws, arrs):
            np.copyto(w, a)
        ths = [threading.Thread(target=one, args=(w,)) for w in ws]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if rep:
            dts.append(time.perf_counter() - t0)
    res["all_cores"] = {"gkeys_per_s": len(ws) * m * len(dts) / sum(dts) / 1e9,
                        "threads": len(ws), "keys_per_thread": m,
                        "timing": "wall clock, best-effort, independent arrays"}
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", default="all")
    ap.add_argument("--min-ms", type=float, default=500.0)
    ap.add_argument("--steps", type=int, default=0)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--n", type=int, default=1 << 24)
    args = ap.parse_args()
    if not O.ref_available():
        print(json.dumps({"unavailable": f"{O.REF_SO} missing (build it with oracle/Makefile "
                                         "where /root/reference exists)"}))
        return
    allowed = set(os.sched_getaffinity(0))
    core, n_allowed, nproc = pin_one_core()
    head = {"kind": "reference", "lib": "oracle/_ref/libnetsort_ref.so", "core": core,
            "cores": 1, "cores_allowed": n_allowed, "nproc": nproc, "cpu": cpu_model(),
            "clock": "CLOCK_PROCESS_CPUTIME_ID (wall alongside)",
            "policy": "restated measure_loop (bench.cpp:39-89): 1 untimed warm-up, untimed "
                      "refill, batches doubling to min_ms of CPU time, cap 2^20"}
    if args.steps:
        head.update(run_steps(args.steps, args.warmup, args.n, allowed))
    else:
        cells = CELLS if args.cells == "all" else args.cells.split(",")
        head["min_ms"] = args.min_ms
        head["cells"] = run_cells(cells, args.min_ms)
    print(json.dumps(head), flush=True)


if __name__ == "__main__":
    main()
