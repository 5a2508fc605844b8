#!/usr/bin/env python
"""bench.py — B200 hybrid network-base-case sort, one JSON line on rank 0.

Workload (BASELINE.json configs[4], the largest single-GPU configuration of
the metric "sorted int32 Gkeys/s at n=10K-1G"): ONE uniform-random int32
array of n = 2^30 keys (values int32(SplitMix64(42).next() >> 33), generated
on the device, identical to the oracle's stream), sorted by merge sort with
the 6To8 network base case.  At N = 1 that is the single-GPU merge sort of
1 G keys; under torchrun with N > 1 the array is sharded evenly and sorted by
the sample sort (local merge sort -> 255 regular samples per GPU -> NCCL
all-gather + all-to-all -> g-way merge): total work fixed, scaling "strong".

  value  : n / (device time of the sort), inputs resident in HBM, CUDA events
           on the launching stream, max over ranks; the input is restored by
           an untimed device copy before every step (4 GiB >> 126 MB L2, so
           no step sees a warm L2 for its input).
  e2e    : the same metric through the public API with HOST buffers: pinned
           int32 numpy array -> optimized_merge_sort(array, 6To8) (C ABI
           ns_merge_sort_host_i32: H2D, sort, D2H, sync) timed by wall clock.
  roofline: dominant kernel (merge_pass_kernel) — algorithmic bytes per
           launch (8 B/key: read + write every key once) / its average launch
           time from the library's own per-launch CUDA events, vs the measured
           HBM copy bandwidth in MEASURED_PEAKS.json.
  cpu_baseline: the reference itself (oracle/_ref, compiled from
           /root/reference) — optimized_merge_sort<int32_t>(6To8) on one core,
           on a 2^24-key sample of the same distribution.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = None
N_DEFAULT = 1 << 30
SEED = 42
GAMMA = 0x9E3779B97F4A7C15


def baseline_metric():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        return json.load(f)["metric"]


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference (oracle/_ref) or the C port (oracle)
# ---------------------------------------------------------------------------
def cpu_baseline(seconds: float = 10.0, n: int = 1 << 24):
    import numpy as np
    from oracle import oracle as O
    a = O.generate_i32("random", n, SEED)
    mask, vs = O.CONFIGS["6To8"]
    if O.ref_available():
        fn = lambda x: O.ref().ref_merge_sort_i32(x, len(x), mask, vs, None)  # noqa: E731
        kind = "reference"
    else:
        fn = lambda x: O.lib().oracle_merge_sort_i32(x, 0, len(x) - 1, mask, vs, None)  # noqa
        kind = "port"
    times = []
    t_total = time.perf_counter()
    while True:
        w = a.copy()
        t0 = time.perf_counter()
        fn(w)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_total > seconds or len(times) >= 8:
            break
    assert np.all(w[:-1] <= w[1:])
    best = min(times)
    return {"value": n / best / 1e9, "unit": "Gkeys/s", "cores": 1, "kind": kind,
            "sample": f"optimized_merge_sort<int32_t>(6To8) on {n} uniform-random keys "
                      f"(seed {SEED}), 1 thread, best of {len(times)} runs",
            "cpu": _cpu_model()}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, metric):
    """--impl reference: the reference's CPU merge sort (oracle/_ref, else the
    oracle port) on the host cores, one independent 2^22-key sample of the
    workload's distribution per thread per step (the reference is
    single-threaded per array, bench.hpp:53-57)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    from oracle import oracle as O
    O.build()
    threads = len(os.sched_getaffinity(0))
    m = 1 << 22
    mask, vs = O.CONFIGS["6To8"]
    if O.ref_available():
        kind = "reference"
        fn = lambda x: O.ref().ref_merge_sort_i32(x, len(x), mask, vs, None)  # noqa: E731
    else:
        kind = "port"
        fn = lambda x: O.lib().oracle_merge_sort_i32(x, 0, len(x) - 1, mask, vs, None)  # noqa
    pristine = [O.generate_i32("random", m, SEED + t) for t in range(threads)]
    work = [p.copy() for p in pristine]

    def step():
        for w, p in zip(work, pristine):
            np.copyto(w, p)
        ths = [threading.Thread(target=fn, args=(w,)) for w in work]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0

    for _ in range(args.warmup):
        step()
    dt = [step() for _ in range(args.steps)]
    for w in work:
        assert np.all(w[:-1] <= w[1:])
    total = sum(dt)
    v = threads * m * args.steps / total / 1e9
    line = {"metric": metric, "value": v, "unit": "Gkeys/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": {"workload": "merge sort 6To8, uniform-random int32 (BASELINE configs[4] "
                                   "distribution), bounded CPU sample",
                       "keys_per_thread_per_step": m, "threads": threads},
            "cpu_baseline": {"value": v, "unit": "Gkeys/s", "cores": threads, "kind": kind,
                             "sample": f"{threads} threads x optimized_merge_sort<int32_t>(6To8) "
                                       f"on independent {m}-key arrays per step",
                             "cpu": _cpu_model()},
            "e2e": {"value": v, "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, metric):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2503_05934_b200 as ns
    from paper_2503_05934_b200 import samplesort
    from paper_2503_05934_b200._lib import check

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_TEST_ONE_GPU=1 (code-path check only, never a bench number): every
    # rank on cuda:0 with gloo metadata collectives, as tests/multiproc_p2p_gpu.py
    one_gpu = os.environ.get("BENCH_TEST_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    def all_reduce(t, op):  # gloo (one-GPU code-path check) reduces host tensors
        if world > 1 and dist.get_backend() == "gloo":
            c = t.cpu()
            dist.all_reduce(c, op=op)
            t.copy_(c)
        elif world > 1:
            dist.all_reduce(t, op=op)

    L = ns.lib()
    cfg = ns.find_config("6To8")
    n = args.n
    m = n // world
    stream = torch.cuda.current_stream().cuda_stream

    keys = torch.empty(m, dtype=torch.int32, device=dev)
    # rank r's shard = positions [r*m, (r+1)*m) of the global SplitMix64 stream
    check(L.ns_generate_i32(keys.data_ptr(), m, 0, (SEED + rank * m * GAMMA) % 2**64, stream),
          "generate")
    pristine = keys.clone()
    d_in = ns.multiset_digest(keys)
    ops = samplesort.DeviceOps(cfg.width_mask, cfg.varsort_max)

    exchange = {"mode": args.exchange}

    def step():
        if world == 1:
            ops.local_sort(keys)
            return keys
        try:
            return samplesort.sample_sort(keys, ops=ops, exchange=exchange["mode"])
        except samplesort.P2PUnavailable as e:  # raised on every rank together
            if exchange["mode"] != "p2p":
                raise
            exchange["mode"] = "nccl"
            exchange["p2p_error"] = str(e)[:200]
            return samplesort.sample_sort(keys, ops=ops, exchange="nccl")

    for _ in range(args.warmup):
        keys.copy_(pristine)
        out = step()
    torch.cuda.synchronize()
    # correctness of the last warm-up step (size-independent properties)
    local_ok = ns.count_inversions(out) == 0
    if world == 1:
        local_ok = local_ok and ns.multiset_digest(out) == d_in

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    launches0 = L.ns_launch_count()
    wall0 = time.perf_counter()
    for i in range(args.steps):
        keys.copy_(pristine)  # untimed restore (outside the events)
        ev[i][0].record()
        out = step()
        ev[i][1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = L.ns_launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    times = [a.elapsed_time(b) for a, b in ev]
    total_ms = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if world > 1:
        all_reduce(total_ms, dist.ReduceOp.MAX)
    total_ms = float(total_ms.item())
    ms_per_step = total_ms / args.steps
    value = n / (ms_per_step * 1e-3) / 1e9

    # one profiled step: per-kernel-class device time from the library's events
    keys.copy_(pristine)
    torch.cuda.synchronize()
    check(L.ns_profile_enable(1), "profile")
    out = step()
    torch.cuda.synchronize()
    import ctypes as C
    prof = {}
    for k in range(L.ns_profile_kinds()):
        t, c = C.c_double(), C.c_uint64()
        check(L.ns_profile_read(k, C.byref(t), C.byref(c)), "profile read")
        if c.value:
            prof[L.ns_profile_kind_name(k).decode()] = {"ms": t.value, "launches": c.value}
    check(L.ns_profile_enable(0), "profile")
    step_prof_ms = sum(v["ms"] for v in prof.values())

    peak, peak_kind = measured_peaks()
    dom = max(prof, key=lambda k: prof[k]["ms"]) if prof else None
    roofline = None
    if dom:
        avg_ms = prof[dom]["ms"] / prof[dom]["launches"]
        bytes_per_launch = 8 * m  # every merge/tile pass reads and writes each key once
        ach = bytes_per_launch / (avg_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(dom, {}).get("dram_bytes_per_launch")
        roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak,
                    "peak_source": peak_kind, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic, "bytes_per_launch": bytes_per_launch,
                    "avg_launch_ms": avg_ms, "launches_per_step": prof[dom]["launches"],
                    "share_of_step": prof[dom]["ms"] / step_prof_ms if step_prof_ms else None}
    # whole-sort byte model: B = 8 n P, P = tile pass + merge passes
    passes = (prof.get("tile_sort", {}).get("launches", 0) +
              prof.get("merge_pass", {}).get("launches", 0))
    model = {"passes": passes, "bytes": 8 * m * passes,
             "frac_all_passes": 8 * m * passes / (ms_per_step * 1e-3) / 1e9 / peak,
             "frac_single_pass_floor": 8 * m / (ms_per_step * 1e-3) / 1e9 / peak}

    # e2e through the public API with host buffers
    e2e = None
    if world == 1:
        host = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        host_src = pristine.cpu().numpy()
        e2e_steps = max(1, min(args.steps, 3))
        dts = []
        ns.optimized_merge_sort(host, cfg)  # warm the C-ABI host cache
        for _ in range(e2e_steps):
            np.copyto(host, host_src)
            t0 = time.perf_counter()
            ns.optimized_merge_sort(host, cfg)
            dts.append(time.perf_counter() - t0)
        assert np.all(host[:-1] <= host[1:])
        e2e = {"value": n * e2e_steps / sum(dts) / 1e9, "unit": "Gkeys/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "path": "optimized_merge_sort(pinned numpy int32, 6To8) -> ns_merge_sort_host_i32",
               "steps": e2e_steps}
        del host, host_src
    else:
        # per rank: H2D of the shard from pinned memory, sample sort, D2H of the result
        hs = pristine.cpu().pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.barrier()
        e0.record()
        keys.copy_(hs, non_blocking=True)
        out = samplesort.sample_sort(keys, ops=ops, exchange=exchange["mode"])
        res = out.cpu()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        all_reduce(t, dist.ReduceOp.MAX)
        e2e = {"value": n / (float(t.item()) * 1e-3) / 1e9, "unit": "Gkeys/s",
               "h2d_bytes_per_step": 4 * m, "d2h_bytes_per_step": 4 * res.numel(),
               "path": "per-rank pinned shard -> sample_sort -> host", "steps": 1}

    # NVLink roofline of the exchange: one step with the
    # sample sort's own phase events.  exchange="p2p" fuses the all-to-all into
    # the first merge round (peer HBM read over NVLink), so the fused phase is
    # the exchange; "nccl" times the all_to_all itself.  Bytes = keys this rank
    # pulls from / sends to its peers; time = max over ranks.
    nvlink = None
    if world > 1:
        tm = samplesort.SampleSortTiming()
        keys.copy_(pristine)
        torch.cuda.synchronize()
        dist.barrier()
        samplesort.sample_sort(keys, ops=ops, exchange=exchange["mode"], timing=tm)
        phase_ms = tm.merge_ms if exchange["mode"] == "p2p" else tm.exchange_ms
        v = torch.tensor([phase_ms, tm.local_sort_ms, float(tm.send_bytes)], dtype=torch.float64,
                         device=dev)
        vmax = v.clone()
        all_reduce(vmax, dist.ReduceOp.MAX)
        peer_gbs = 770.0  # measured peer copy per direction (B200_PROFILING.md)
        per_rank_bytes = float(vmax[2].item())
        ach = per_rank_bytes / (float(vmax[0].item()) * 1e-3) / 1e9 if vmax[0] > 0 else None
        nvlink = {"phase": "pull-merge (fused all-to-all)" if exchange["mode"] == "p2p"
                  else "nccl all_to_all", "phase_ms_max": float(vmax[0].item()),
                  "local_sort_ms_max": float(vmax[1].item()),
                  "bytes_per_rank_max": per_rank_bytes, "achieved_gbs": ach,
                  "peak_gbs": peer_gbs, "peak_source": "measured peer copy (fallback figure)",
                  "frac": (ach / peer_gbs) if ach else None}

    ok = torch.tensor([1 if local_ok else 0], device=dev)
    if world > 1:
        all_reduce(ok, dist.ReduceOp.MIN)

    line = {"metric": metric, "value": value, "unit": "Gkeys/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic",
            "config": {"workload": ("merge sort 6To8" if world == 1 else
                                    "sample sort (local merge sort 6To8 + " +
                                    ("pull-merge over NVLink peer memory)"
                                     if exchange["mode"] == "p2p" else "NCCL all-to-all)")) +
                       f", one uniform-random int32 array, n={n} (BASELINE configs[4])",
                       "n": n, "keys_per_gpu": m, "distribution": "uniform [0, 2^31), seed 42",
                       "parallelism": "replicas/shards over NCCL" if world > 1 else "single GPU",
                       "l2": f"input {4 * n / 2**30:.2f} GiB vs 126 MB L2; restored by an "
                             "untimed D2D copy before each step"},
            "exchange": exchange if world > 1 else None,
            "gpu_launches": int(launches), "wall_ms_timed_region": wall * 1e3,
            "roofline": roofline, "byte_model": model, "kernel_profile": prof,
            "e2e": e2e, "clocks": clk, "verified": bool(ok.item())}
    if nvlink is not None:
        line["nvlink"] = nvlink
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    if rank == 0 and world == 1 and not args.no_size_sweep:
        line["size_sweep"] = size_sweep(ns, L, dev, peak)
    if rank == 0 and world == 1 and not args.no_batch:
        line["base_case_batch"] = base_case_batch(ns, L, dev, peak)
    if rank == 0 and world == 1 and args.extra:
        line["other_configs"] = other_configs(ns, L, dev)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def base_case_batch(ns, L, dev, peak):
    """BASELINE configs[1], the base-case kernel alone: 2^24 independent int32
    arrays, lengths uniform in {3..8}, packed with a uint32 offsets array,
    each sorted by its size-specific network.  Kernel time from the library's
    own launch events (median of 7; the call adds one 4-byte validation
    read-back), algorithmic bytes 8 per key + 4 per offset, checked against
    the oracle (the checker only)."""
    import ctypes as C
    import numpy as np
    import torch
    from paper_2503_05934_b200._lib import check
    from oracle import oracle as O
    offs, keys = O.generate_batch_i32(1 << 24, SEED)
    k = torch.from_numpy(keys).to(dev)
    o = torch.from_numpy(offs.view("int32")).to(dev)
    w = k.clone()
    ns.sort_small_batch(w, o)
    ok = bool(np.array_equal(w.cpu().numpy(), O.sort_small_batch(keys, offs)))
    ts = []
    for _ in range(7):
        w.copy_(k)
        torch.cuda.synchronize()
        check(L.ns_profile_enable(1), "profile")
        ns.sort_small_batch(w, o)
        torch.cuda.synchronize()
        tot = 0.0
        for kind in range(L.ns_profile_kinds()):
            t, c = C.c_double(), C.c_uint64()
            check(L.ns_profile_read(kind, C.byref(t), C.byref(c)), "profile read")
            tot += t.value
        check(L.ns_profile_enable(0), "profile")
        ts.append(tot)
    ms = statistics.median(ts)
    nbytes = 8 * len(keys) + 4 * len(offs)
    gbs = nbytes / (ms * 1e-3) / 1e9
    return {"workload": "BASELINE configs[1]: 2^24 ragged int32 arrays, lengths U{3..8}, "
                        "uint32 offsets, size-specific networks",
            "num_arrays": 1 << 24, "num_keys": int(len(keys)), "kernel_ms": ms,
            "gkeys_per_s": len(keys) / (ms * 1e-3) / 1e9, "bytes": nbytes,
            "achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak, "verified": ok}


def size_sweep(ns, L, dev, peak):
    """The metric across the range BASELINE.json names (n = 10K..1G): merge
    sort 6To8 of uniform-random keys at each n, device time by CUDA-graph
    replay (sort + an untimed-by-subtraction input restore), with the byte
    model's fraction (8n bytes per pass, 1 tile pass + ceil(log2(n/T)) merge
    passes, T = the library's tile: 16384 keys from 2^21, else 8192) of the
    measured HBM bandwidth.  Below ~2^24 keys the data
    is L2-resident and the sort is latency-bound: the fraction is reported,
    not a bandwidth statement.  2^30 is the headline line itself."""
    import torch
    from paper_2503_05934_b200._lib import check
    out = {}
    s = torch.cuda.current_stream().cuda_stream
    cfg = ns.find_config("6To8")
    for n in (10_000, 100_000, 1_000_000, 1 << 22, 1 << 24, 1 << 26, 1 << 28):
        src = torch.empty(n, dtype=torch.int32, device=dev)
        check(L.ns_generate_i32(src.data_ptr(), n, 0, SEED, s), "generate")
        w = src.clone()
        fn = lambda: ns.optimized_merge_sort(w, cfg)  # noqa: E731
        restore = lambda: w.copy_(src)  # noqa: E731
        reps = max(3, min(50, (1 << 26) // n))
        for _ in range(3):
            restore()
            fn()
        torch.cuda.synchronize()
        times = []
        for body in ((restore, fn), (restore,)):
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for f in body:
                    f()
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b) / reps)
        ms = max(times[0] - times[1], 1e-6)
        restore()
        fn()
        tile_lg = 14 if n >= (1 << 21) else 13  # the library's int32 tile (16384 / 8192)
        passes = 1 + max(0, (n - 1).bit_length() - tile_lg)
        out[str(n)] = {"ms": ms, "gkeys_per_s": n / (ms * 1e-3) / 1e9,
                       "frac_all_passes": 8 * n * passes / (ms * 1e-3) / 1e9 / peak,
                       "sorted": ns.count_inversions(w) == 0}
        del src, w
    ns.release_scratch()
    torch.cuda.empty_cache()
    return out


def other_configs(ns, L, dev):
    """The other BASELINE configs.  Merge sort (no host round trip inside) is
    timed as a CUDA-graph replay of the C-ABI call, i.e. pure device time with
    the input restored inside the graph by a D2D copy whose own time is
    subtracted; quick sort and the batch (one D2H read each by design) are
    timed per call with CUDA events on the stream (host round trip included)
    and also reported as the sum of their kernels' device time from the
    library's per-launch events."""
    import ctypes as C
    import torch
    from paper_2503_05934_b200._lib import check
    from oracle import oracle as O
    res = {}
    s = torch.cuda.current_stream().cuda_stream

    def kernel_ms(fn, restore):
        restore()
        fn()  # warm: lazy module loading and smem attributes stay out of the profile
        restore()
        torch.cuda.synchronize()
        check(L.ns_profile_enable(1), "profile")
        fn()
        torch.cuda.synchronize()
        tot = 0.0
        for k in range(L.ns_profile_kinds()):
            t, c = C.c_double(), C.c_uint64()
            check(L.ns_profile_read(k, C.byref(t), C.byref(c)), "profile read")
            tot += t.value
        check(L.ns_profile_enable(0), "profile")
        return tot

    def call_ms(fn, restore, reps=10):
        for _ in range(3):
            restore()
            fn()
        ts = []
        for _ in range(reps):
            restore()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    def graph_ms(fn, restore, reps=20):
        for _ in range(3):
            restore()
            fn()
        torch.cuda.synchronize()
        g_full, g_copy = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
        with torch.cuda.graph(g_full):
            restore()
            fn()
        with torch.cuda.graph(g_copy):
            restore()
        out = []
        for g in (g_full, g_copy):
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(reps):
                g.replay()
            b.record()
            torch.cuda.synchronize()
            out.append(a.elapsed_time(b) / reps)
        return max(out[0] - out[1], 1e-6)

    def single(name, algo, cfgname, dist, n, key="i32"):
        gen = O.generate_i32 if key == "i32" else O.generate_i64
        a = torch.from_numpy(gen(dist, n, SEED)).to(dev)
        w = a.clone()
        cfg = ns.find_config(cfgname)
        fn = lambda: (ns.optimized_merge_sort if algo == "merge"  # noqa: E731
                      else ns.optimized_quick_sort)(w, cfg)
        restore = lambda: w.copy_(a)  # noqa: E731
        rec = {"n": n, "kernel_ms": kernel_ms(fn, restore), "call_ms": call_ms(fn, restore)}
        if algo == "merge":
            rec["graph_ms"] = graph_ms(fn, restore)
            rec["gkeys_per_s"] = n / (rec["graph_ms"] * 1e-3) / 1e9
        else:
            rec["gkeys_per_s"] = n / (rec["call_ms"] * 1e-3) / 1e9
        w.copy_(a)
        fn()
        rec["sorted"] = ns.count_inversions(w) == 0
        if key == "i64":
            rec["key"] = "int64 (the reference's own benchmark type, full 64-bit values)"
            if algo == "merge" and n > (1 << 14):
                # byte model: 16 B per key per pass (one tile pass + one pass
                # per doubling from the 8192-key tile)
                passes = 1 + max(0, (n - 1).bit_length() - 13)
                rec["hbm_frac_all_passes"] = 16 * n * passes / (rec["graph_ms"] * 1e-3) / 1e9 \
                    / measured_peaks()[0]
        res[name] = rec

    single("ms_6to8_random_10k", "merge", "6To8", "random", 10_000)
    for n in (25_000, 100_000, 1_000_000):
        for d in ("random", "sorted", "nearly_sorted"):
            single(f"ms_6to8_{d}_{n}", "merge", "6To8", d, n)
    for n in (10_000, 1_000_000, 16_777_216):
        for d in ("sorted", "random"):
            single(f"qs_3to5_{d}_{n}", "quick", "3To5", d, n)
    # int64 keys
    for n in (1_000_000, 1 << 28):
        single(f"ms_6to8_random_i64_{n}", "merge", "6To8", "random", n, key="i64")
    for n in (1_000_000, 16_777_216):
        single(f"qs_3to5_random_i64_{n}", "quick", "3To5", "random", n, key="i64")
    torch.cuda.empty_cache()
    # stable key-value sort (int32 keys + 4-byte payload), SURVEY.md §8(f) row 4
    n = 1 << 26
    kk = torch.from_numpy(O.generate_i32("random", n, SEED)).to(dev)
    vv = torch.arange(n, dtype=torch.int32, device=dev)
    wk, wv = kk.clone(), vv.clone()
    fn = lambda: ns.sort_pairs(wk, wv)  # noqa: E731
    restore = lambda: (wk.copy_(kk), wv.copy_(vv))  # noqa: E731
    ms = graph_ms(fn, restore, reps=5)
    res["sort_pairs_i32_random_2^26"] = {"n": n, "graph_ms": ms,
                                         "gkeys_per_s": n / (ms * 1e-3) / 1e9}
    del kk, vv, wk, wv
    torch.cuda.empty_cache()
    # base-case batch, 2^24 ragged arrays
    offs, keys = O.generate_batch_i32(1 << 24, SEED)
    k = torch.from_numpy(keys).to(dev)
    o = torch.from_numpy(offs.view("int32")).to(dev)
    w = k.clone()
    fn = lambda: ns.sort_small_batch(w, o)  # noqa: E731
    restore = lambda: w.copy_(k)  # noqa: E731
    kms, cms = kernel_ms(fn, restore), call_ms(fn, restore)
    nbytes = 8 * len(keys) + 4 * len(offs)
    res["base_case_batch_2^24"] = {"num_arrays": 1 << 24, "num_keys": int(len(keys)),
                                   "kernel_ms": kms, "call_ms": cms,
                                   "gkeys_per_s": len(keys) / (cms * 1e-3) / 1e9,
                                   "kernel_hbm_gbs": nbytes / (kms * 1e-3) / 1e9}
    # segmented quick sort 65536 x 16384
    n = 65536 * 16384
    seg = torch.empty(n, dtype=torch.int32, device=dev)
    check(L.ns_generate_i32(seg.data_ptr(), n, 0, SEED, s), "generate")
    w = seg.clone()
    cfg = ns.find_config("3To5")
    fn = lambda: ns.segmented_sort(w, 16384, cfg, ns.Algorithm.quick_sort)  # noqa: E731
    restore = lambda: w.copy_(seg)  # noqa: E731
    ms = graph_ms(fn, restore, reps=5)
    res["qs_3to5_segmented_65536x16384"] = {"n": n, "graph_ms": ms,
                                            "gkeys_per_s": n / (ms * 1e-3) / 1e9,
                                            "hbm_gbs": 8 * n / (ms * 1e-3) / 1e9}
    del seg, w
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--keys", "--n", dest="n", type=int, default=N_DEFAULT,
                    help="total keys (--keys under torchrun: its parser claims --n)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--extra", action="store_true", help="also time the other BASELINE configs")
    ap.add_argument("--no-batch", action="store_true",
                    help="skip the base-case batch kernel (BASELINE configs[1]) object")
    ap.add_argument("--no-size-sweep", action="store_true",
                    help="skip the n = 10K..256M merge-sort sweep (N=1 only)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="p2p",
                    help="N>1: pull-merge over peer memory (default) or NCCL all-to-all")
    args = ap.parse_args()
    metric = baseline_metric()
    if args.impl == "reference":
        run_reference(args, metric)
    else:
        run_ours(args, metric)


if __name__ == "__main__":
    main()
