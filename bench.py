#!/usr/bin/env python
"""bench.py — B200 hybrid network-base-case sort, one JSON line on rank 0.

Headline workload (BASELINE.json configs[4], the largest single-GPU
configuration of the metric "sorted int32 Gkeys/s at n=10K-1G"): ONE
uniform-random int32 array of n = 2^30 keys (int32(SplitMix64(42).next() >>
33), generated on the device), merge sort with the 6To8 network base case.
Under torchrun with N > 1 the same array is sharded evenly and sample-sorted
(local merge sort -> 255 regular samples per GPU -> splitters -> all-to-all
over NVLink -> g-way merge): total work fixed, scaling "strong".

  value   : n / device time of the sort (CUDA events on the launching stream,
            max over ranks), inputs resident in HBM; the input is restored by
            an untimed D2D copy before every step (4 GiB >> 126 MB L2).
  e2e     : the same metric through the public API with HOST buffers (pinned
            numpy array -> optimized_merge_sort -> ns_merge_sort_host_i32:
            H2D, sort, D2H, sync), wall clock.
  roofline: the dominant kernel's algorithmic bytes per launch (8 B/key) over
            its average launch time (the library's per-launch CUDA events),
            vs the measured HBM bandwidth in MEASURED_PEAKS.json.
  configs : every other BASELINE cell (configs[0..3]: MS 6To8 at 10K, 25K /
            100K / 1M x random / sorted / nearly sorted, QS 3To5 at 10K / 1M /
            16M x sorted / random, the 2^24-array base-case batch, the
            65,536 x 16,384 segmented batch): device time, byte-model fraction,
            verification against SHA-256 digests of the REFERENCE's own sorted
            output (tests/golden/golden.json), e2e at 10K and 1M, and the
            reference's time on ONE pinned core for the same input.
  cpu_baseline / --impl reference: the reference itself (oracle/_ref, built
            from /root/reference by oracle/Makefile) on one pinned core in a
            child process (oracle/cpu_ref_bench.py), CPU time with the
            reference harness's doubling-batch policy (bench.cpp:39-89).

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
        self.lines = []   # (host time the sample arrived, csv line)
        self.t0 = None

    def launch(self):
        """Starts nvidia-smi (its start-up takes ~100 ms: call this before the
        timed region); only samples that arrive between start() and stop() count."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def start(self):
        if self.proc is None:
            self.launch()
        self.t0 = time.time()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        time.sleep(0.03)  # the sample taken at the end of the region is still in the pipe
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        inside = [ln for (t, ln) in self.lines if self.t0 is not None and self.t0 <= t <= t1 + 0.03]
        for ln in (inside if inside else [ln for (_, ln) in self.lines]):
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
# CPU arm: the reference (oracle/_ref) on ONE pinned core, in a child process
# (oracle/cpu_ref_bench.py: CLOCK_PROCESS_CPUTIME_ID, the reference harness's
# doubling-batch policy restated at int32, bench.cpp:39-89)
# ---------------------------------------------------------------------------
def cpu_child(extra, timeout=900):
    cmd = [sys.executable, os.path.join(ROOT, "oracle", "cpu_ref_bench.py")] + extra
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
        lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
        if r.returncode != 0 or not lines:
            return {"unavailable": f"cpu_ref_bench rc={r.returncode}: {r.stderr[-300:]}"}
        return json.loads(lines[-1])
    except Exception as e:  # noqa: BLE001 - reported in the line
        return {"unavailable": f"cpu_ref_bench failed: {e!r}"[:300]}


HEADLINE_CPU_CELL = "merge:6To8:random:16777216"


def cpu_baseline_from(cells):
    """cpu_baseline object of the headline: the reference's merge sort 6To8 on
    a 2^24-key uniform-random sample of the 2^30 workload, one pinned core."""
    if "cells" not in cells or HEADLINE_CPU_CELL not in cells["cells"]:
        return {"value": None, "unit": "Gkeys/s", "cores": 1, "kind": "reference",
                "sample": "unavailable", "detail": cells.get("unavailable")}
    c = cells["cells"][HEADLINE_CPU_CELL]
    return {"value": c["gkeys_per_s"], "unit": "Gkeys/s", "cores": 1, "kind": "reference",
            "sample": "optimized_merge_sort<int32_t>(6To8) from oracle/_ref (the reference "
                      "compiled from its own sources) on a 2^24-key uniform-random sample "
                      f"(seed {SEED}) of the 2^30 workload; {c['iterations']} timed call(s) "
                      f"after one untimed warm-up, CPU time {c['cpu_ms']:.1f} ms per call "
                      f"(wall {c['wall_ms']:.1f} ms); a 2^30 array would take ~27/21 of the "
                      "per-key time (merge levels), so this overstates the CPU",
            "core": cells.get("core"), "nproc": cells.get("nproc"), "cpu": cells.get("cpu"),
            "clock": cells.get("clock")}


def workload_config(n, world, exchange):
    return {"workload": ("merge sort 6To8" if world == 1 else
                         "sample sort (local merge sort 6To8 + " +
                         ("pull-merge over NVLink peer memory)" if exchange == "p2p"
                          else "NCCL all-to-all)")) +
                        f", one uniform-random int32 array, n={n} (BASELINE configs[4])",
            "n": n, "keys_per_gpu": n // world, "distribution": "uniform [0, 2^31), seed 42",
            "parallelism": "shards over NCCL/NVLink" if world > 1 else "single GPU",
            "l2": f"input {4 * n / 2**30:.2f} GiB vs 126 MB L2; restored by an untimed D2D "
                  "copy before each step"}


def run_reference(args, metric):
    """--impl reference: the reference's own CPU merge sort (oracle/_ref) on
    ONE pinned core — its path is single-threaded (bench.hpp:53-57) — each
    step a 2^24-key uniform-random sample of the 2^30 workload, CPU time per
    call.  An all-cores figure (independent arrays, one per core) is reported
    beside it as all_cores_not_reference_path.  Under torchrun only rank 0
    runs."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    m = 1 << 24
    r = cpu_child(["--steps", str(args.steps), "--warmup", str(args.warmup), "--n", str(m)],
                  timeout=1800)
    if "unavailable" in r:
        print(json.dumps({"impl": "reference", "unavailable": r["unavailable"]}), flush=True)
        return
    ms = r["cpu_ms_per_step"]
    v = m / (ms * 1e-3) / 1e9
    line = {"metric": metric, "value": v, "unit": "Gkeys/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": workload_config(args.n, world, args.exchange),
            "cpu_baseline": {"value": v, "unit": "Gkeys/s", "cores": 1, "kind": "reference",
                             "sample": f"each step: optimized_merge_sort<int32_t>(6To8) from "
                                       f"oracle/_ref on a {m}-key uniform-random sample of the "
                                       f"workload, one pinned core, CPU time "
                                       f"(CLOCK_PROCESS_CPUTIME_ID), refill untimed",
                             "core": r.get("core"), "nproc": r.get("nproc"), "cpu": r.get("cpu"),
                             "wall_ms_per_step": r.get("wall_ms_per_step")},
            "e2e": {"value": v, "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0},
            "all_cores_not_reference_path": r.get("all_cores")}
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
    # correctness of the last warm-up step (size-independent properties):
    # every rank's slice sorted, the ranks' slices in order across rank
    # boundaries, and the multiset of all output keys == that of all input
    # keys (sum and xor of mix64(key), combined over ranks)
    local_ok = ns.count_inversions(out) == 0
    d_out = ns.multiset_digest(out) if out.numel() else (0, 0)
    if world == 1:
        local_ok = local_ok and d_out == d_in
    else:
        import numpy as _np
        cnt = out.numel()
        mine = torch.tensor([cnt, int(out[0]) if cnt else 0, int(out[-1]) if cnt else 0,
                             d_in[0] - 2**63, d_in[1] - 2**63, d_out[0] - 2**63,
                             d_out[1] - 2**63], dtype=torch.int64)
        parts = [torch.empty_like(mine) for _ in range(world)]
        if dist.get_backend() == "gloo":
            dist.all_gather(parts, mine)
        else:
            pd = [p.to(dev) for p in parts]
            dist.all_gather(pd, mine.to(dev))
            parts = [p.cpu() for p in pd]
        rows = [[int(x) for x in p.tolist()] for p in parts]
        u = lambda v: (v + 2**63) % 2**64  # noqa: E731
        sin = sum(u(r[3]) for r in rows) % 2**64
        sout = sum(u(r[5]) for r in rows) % 2**64
        xin = xout = 0
        for r in rows:
            xin ^= u(r[4])
            xout ^= u(r[6])
        nonempty = [r for r in rows if r[0] > 0]
        order_ok = all(a[2] <= b[1] for a, b in zip(nonempty, nonempty[1:]))
        count_ok = sum(r[0] for r in rows) == n
        local_ok = local_ok and sin == sout and xin == xout and order_ok and count_ok
        del _np

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    clocks = Clocks(local)
    clocks.launch()  # nvidia-smi starts up outside the timed region
    time.sleep(0.15)
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
        # a stream of K sorts of the 2^30-key pinned host array through the
        # stream-ordered host API (ns_merge_sort_host_async_i32): every step
        # uploads its input, sorts and downloads the result; two streams, so
        # step k+1's upload overlaps step k's download (PCIe is full duplex)
        host_in = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy()
        np.copyto(host_in, pristine.cpu().numpy())
        outs = [torch.empty(n, dtype=torch.int32, pin_memory=True).numpy() for _ in range(2)]
        sts = [torch.cuda.Stream(), torch.cuda.Stream()]
        for j in range(2):  # warm: allocates each stream's device buffers
            ns.sort_host_async(host_in, outs[j], cfg, stream=sts[j])
        torch.cuda.synchronize()
        e2e_steps = max(2, min(args.steps, 10))
        t0 = time.perf_counter()
        for k in range(e2e_steps):
            ns.sort_host_async(host_in, outs[k % 2], cfg, stream=sts[k % 2])
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        for o in outs:
            assert np.all(o[:-1] <= o[1:])
        # one blocking call (the reference's own call shape, optimized_merge_sort
        # on a pinned host array) for the single-sort latency
        host = outs[0]
        np.copyto(host, host_in)
        t1 = time.perf_counter()
        ns.optimized_merge_sort(host, cfg)
        single = time.perf_counter() - t1
        assert np.all(host[:-1] <= host[1:])
        e2e = {"value": n * e2e_steps / dt / 1e9, "unit": "Gkeys/s",
               "h2d_bytes_per_step": 4 * n, "d2h_bytes_per_step": 4 * n,
               "path": "sort_host_async(pinned numpy in -> pinned numpy out, 6To8) -> "
                       "ns_merge_sort_host_async_i32, steps alternating two streams (each "
                       "step's H2D + sort + D2H inside the wall-clock region; step k+1's "
                       "upload overlaps step k's download)",
               "steps": e2e_steps,
               "single_call": {"value": n / single / 1e9, "unit": "Gkeys/s",
                               "path": "optimized_merge_sort(pinned numpy int32, 6To8) -> "
                                       "ns_merge_sort_host_i32 (blocking; H2D overlapped "
                                       "with chunk sorts)"}}
        del host_in, outs, host
        ns.release_scratch()  # frees the host-API device caches too (ns_release_cache)
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
            "config": workload_config(n, world, exchange["mode"]),
            "exchange": exchange if world > 1 else None,
            "gpu_launches": int(launches), "wall_ms_timed_region": wall * 1e3,
            "roofline": roofline, "byte_model": model, "kernel_profile": prof,
            "e2e": e2e, "clocks": clk, "verified": bool(ok.item())}
    if nvlink is not None:
        line["nvlink"] = nvlink
    if world > 1 and not args.no_configs:
        sb = sharded_batches(ns, L, dev, world, rank, all_reduce)
        if rank == 0:
            line["sharded_batches"] = sb
    if rank == 0 and world == 1 and not args.no_size_sweep:
        line["size_sweep"] = size_sweep(ns, L, dev, peak)
    if rank == 0 and world == 1 and not args.no_configs:
        line["configs"] = all_configs(ns, L, dev, peak)
    if rank == 0 and world == 1 and args.extra:
        line["other_configs"] = other_configs(ns, L, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cells = cpu_child(["--cells", "all"])
        line["cpu_baseline"] = cpu_baseline_from(cells)
        if "configs" in line:
            attach_cpu(line["configs"], cells)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# Under torchrun: the two batch configs sharded by array over the ranks
# (independent arrays, no collective on the data path).
# Total work is fixed (the 2^24-array batch, the 65,536 x 16,384 segmented
# batch), each rank sorts its own contiguous share; time = max over ranks.
# ---------------------------------------------------------------------------
def sharded_batches(ns, L, dev, world, rank, all_reduce):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2503_05934_b200 import multigpu

    def timed(fn, restore, reps=3):
        restore()
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            restore()  # untimed
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        t = torch.tensor([min(ts)], dtype=torch.float64, device=dev)
        all_reduce(t, dist.ReduceOp.MAX)
        return float(t.item())

    out = {"scaling": "strong (fixed total work, arrays / segments split over the ranks)"}
    # base-case batch: key-balanced contiguous array ranges (ns_shard_batch_plan)
    offs, keys = ns.generate_batch(1 << 24, SEED)
    ab = multigpu.shard_batch_plan(offs, world)
    a0, a1 = int(ab[rank]), int(ab[rank + 1])
    k0, k1 = int(offs[a0]), int(offs[a1])
    my_offs = (offs[a0:a1 + 1].astype(np.int64) - k0).astype(np.uint32)
    src = torch.from_numpy(keys[k0:k1].copy()).to(dev)
    o = torch.from_numpy(my_offs.view(np.int32)).to(dev)
    w = src.clone()
    st = torch.zeros(1, dtype=torch.int32, device=dev)

    ms = timed(lambda: ns.sort_small_batch(w, o, status=st), lambda: w.copy_(src))
    got = w.cpu().numpy()
    arr = np.repeat(np.arange(a1 - a0), np.diff(my_offs.astype(np.int64)))
    want = keys[k0:k1][np.lexsort((keys[k0:k1], arr))]  # checker: per-array sort
    ok = int(st.item()) == 0 and np.array_equal(got, want)
    okt = torch.tensor([1 if ok else 0], dtype=torch.int32, device=dev)
    all_reduce(okt, dist.ReduceOp.MIN)
    out["batch"] = {"num_arrays": 1 << 24, "num_keys": int(len(keys)), "ms_max_over_ranks": ms,
                    "gkeys_per_s": len(keys) / (ms * 1e-3) / 1e9, "verified": bool(okt.item()),
                    "timing": "CUDA events around the call, best of 3, max over ranks"}
    del keys, offs
    # segmented batch: 65,536 / world whole segments of 16,384 keys per rank
    seg, nseg_total = 16384, 65536
    nseg = nseg_total // world
    m = nseg * seg
    x = torch.empty(m, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream().cuda_stream
    L.ns_generate_i32(x.data_ptr(), m, 0, (SEED + rank * m * GAMMA) % 2**64, stream)
    d_in = ns.multiset_digest(x)
    y = x.clone()
    cfg = ns.find_config("3To5")

    ms2 = timed(lambda: ns.segmented_sort(y, seg, cfg, ns.Algorithm.quick_sort), lambda: y.copy_(x))
    v = y.view(nseg, seg)
    ok2 = bool((v[:, 1:] >= v[:, :-1]).all().item()) and ns.multiset_digest(y) == d_in
    okt = torch.tensor([1 if ok2 else 0], dtype=torch.int32, device=dev)
    all_reduce(okt, dist.ReduceOp.MIN)
    out["segmented"] = {"segments": nseg_total, "seg_len": seg, "ms_max_over_ranks": ms2,
                        "gkeys_per_s": nseg_total * seg / (ms2 * 1e-3) / 1e9,
                        "verified": bool(okt.item()),
                        "timing": "CUDA events around the call, best of 3, max over ranks"}
    del x, y
    return out


# ---------------------------------------------------------------------------
# BASELINE configs[0..3] (configs[4] is the headline): every cell timed on the
# device, checked against the REFERENCE's own sorted output (SHA-256 digests in
# tests/golden/golden.json, made from oracle/_ref by tests/golden/make_golden.py),
# with its byte model and, after the CPU child has run, the reference's
# 1-core time on the same input.
# ---------------------------------------------------------------------------
QS_GRAPH_SAFE = True      # quick sort is planned on the device (no host sync)
BATCH_GRAPH_SAFE = True   # the async batch call writes its status to a device word


def _golden():
    with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
        return json.load(f)


def _sha(a):
    import hashlib
    import numpy as np
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _profile(L, fn):
    """Per-kind (device ms, launches) of one call, from the library's events."""
    import ctypes as C
    import torch
    from paper_2503_05934_b200._lib import check
    torch.cuda.synchronize()
    check(L.ns_profile_enable(1), "profile")
    fn()
    torch.cuda.synchronize()
    out = {}
    for k in range(L.ns_profile_kinds()):
        t, c = C.c_double(), C.c_uint64()
        check(L.ns_profile_read(k, C.byref(t), C.byref(c)), "profile read")
        if c.value:
            out[L.ns_profile_kind_name(k).decode()] = {"ms": t.value, "launches": c.value}
    check(L.ns_profile_enable(0), "profile")
    return out


def device_ms(fn, restore, graph_safe, reps):
    """Device time of one call: CUDA-graph replay of (restore; call) minus
    replay of (restore) when the call is stream-ordered without host syncs,
    else CUDA events around each call (host round trips inside the call are
    then part of the time).  Median-free mean over `reps` replays."""
    import statistics as st
    import torch
    for _ in range(3):
        restore()
        fn()
    torch.cuda.synchronize()
    if graph_safe:
        out = []
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
            out.append(a.elapsed_time(b) / reps)
            del g
        return max(out[0] - out[1], 1e-6), "cuda-graph replay, restore copy subtracted"
    ts = []
    for _ in range(reps):
        restore()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return st.median(ts), "CUDA events per call (median; host round trips inside the call count)"


def e2e_ms(fn_host, src, reps=20):
    """The reference's call shape: a pageable host numpy array sorted in place
    through the public API (H2D, sort, D2H, sync inside), wall clock, median."""
    import statistics as st
    import numpy as np
    w = src.copy()
    for _ in range(3):
        np.copyto(w, src)
        fn_host(w)
    ts = []
    for _ in range(reps):
        np.copyto(w, src)
        t0 = time.perf_counter()
        fn_host(w)
        ts.append((time.perf_counter() - t0) * 1e3)
    return st.median(ts), w


def all_configs(ns, L, dev, peak):
    import numpy as np
    import torch
    gold = _golden()
    gcase = {(c["algo"], c["config"], c["dist"], c["n"]): c["output_sha256"]
             for c in gold["cases"]}
    res = {}

    def single(cell, algo, cfgname, dist, n, e2e=False):
        a = ns.generate(dist, n, SEED)
        d = torch.from_numpy(a).to(dev)
        w = d.clone()
        cfg = ns.find_config(cfgname)
        sort = ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort
        fn = lambda: sort(w, cfg)  # noqa: E731
        restore = lambda: w.copy_(d)  # noqa: E731
        reps = max(5, min(50, (1 << 26) // n))
        ms, how = device_ms(fn, restore, algo == "merge" or QS_GRAPH_SAFE, reps)
        restore()
        prof = _profile(L, fn)
        got = w.cpu().numpy()
        rec = {"config": cfgname, "algorithm": algo, "dist": dist, "n": n, "device_ms": ms,
               "timing": how, "gkeys_per_s": n / (ms * 1e-3) / 1e9,
               "verified": _sha(got) == gcase.get((algo, cfgname, dist, n)),
               "verified_against": "SHA-256 of the reference's sorted output (golden.json)",
               "kernel_launches": int(sum(v["launches"] for v in prof.values())),
               "kernel_profile": prof}
        if algo == "merge":
            passes = (prof.get("tile_sort", {}).get("launches", 0) +
                      prof.get("merge_pass", {}).get("launches", 0))
            nbytes = 8 * n * passes
            rec["byte_model"] = f"8n x {passes} passes (tile sort + merge passes)"
        else:
            lv = prof.get("qs_count", {}).get("launches", 0)
            nbytes = 12 * n * lv + 8 * n
            rec["byte_model"] = (f"{lv} partition level(s) x (count 4n + scatter 8n) + "
                                 "8n bucket sorts (upper bound: every level over all n keys)")
        rec["model_bytes"] = nbytes
        rec["hbm_frac"] = nbytes / (ms * 1e-3) / 1e9 / peak
        rec["l2_resident"] = 8 * n < 100 * 2**20
        if e2e:
            host = ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort
            ems, hw = e2e_ms(lambda x: host(x, cfg), a)
            rec["e2e"] = {"ms": ems, "gkeys_per_s": n / (ems * 1e-3) / 1e9,
                          "path": f"optimized_{algo}_sort(pageable numpy int32, {cfgname}) -> "
                                  f"ns_{algo}_sort_host_i32", "h2d_bytes": 4 * n,
                          "d2h_bytes": 4 * n, "verified": bool(np.array_equal(hw, got))}
        res[cell] = rec
        del d, w

    single("merge:6To8:random:10000", "merge", "6To8", "random", 10_000, e2e=True)
    for n in (25_000, 100_000, 1_000_000):
        for dist in ("random", "sorted", "nearly_sorted"):
            single(f"merge:6To8:{dist}:{n}", "merge", "6To8", dist, n,
                   e2e=(n == 1_000_000 and dist == "random"))
    for n in (10_000, 1_000_000, 16_777_216):
        for dist in ("sorted", "random"):
            single(f"quick:3To5:{dist}:{n}", "quick", "3To5", dist, n,
                   e2e=(n <= 1_000_000))
    torch.cuda.empty_cache()

    # configs[1]: the base-case kernel alone, 2^24 ragged arrays
    b = gold["batch"]
    offs, keys = ns.generate_batch(1 << 24, SEED)
    k = torch.from_numpy(keys).to(dev)
    o = torch.from_numpy(offs.view(np.int32)).to(dev)
    w = k.clone()
    st = torch.ones(1, dtype=torch.int32, device=dev)
    fn = lambda: ns.sort_small_batch(w, o, status=st)  # noqa: E731
    restore = lambda: w.copy_(k)  # noqa: E731
    ms, how = device_ms(fn, restore, BATCH_GRAPH_SAFE, 10)
    restore()
    prof = _profile(L, fn)
    kms = prof.get("sort_small_batch", {}).get("ms")
    nbytes = 8 * len(keys) + 4 * len(offs)
    res["batch:6To8:random:16777216"] = {
        "workload": "BASELINE configs[1]: 2^24 ragged int32 arrays, lengths U{3..8}, uint32 "
                    "offsets, each sorted by its size-specific network",
        "num_arrays": 1 << 24, "num_keys": int(len(keys)), "device_ms": ms, "timing": how,
        "kernel_ms": kms, "gkeys_per_s": len(keys) / (ms * 1e-3) / 1e9, "model_bytes": nbytes,
        "byte_model": "8 B per key (read + write) + 4 B per offset (the validation pass re-reads "
                      "the offsets; not counted)",
        "hbm_frac": nbytes / (ms * 1e-3) / 1e9 / peak,
        "kernel_hbm_frac": nbytes / (kms * 1e-3) / 1e9 / peak if kms else None,
        "verified": _sha(w.cpu().numpy()) == b["output_sha256"] and int(st.item()) == 0,
        "verified_against": "SHA-256 of the reference's sort_small output (golden.json)",
        "path": "ns_sort_small_batch_async_i32 (validation and network phases in one cooperative kernel, no host sync)"}
    del k, o, w
    torch.cuda.empty_cache()

    # configs[3] segmented: 65,536 x 16,384 uniform-random keys (one 2^30 stream)
    g = gold["segmented"]
    nseg, seg = g["full_num_segments"], g["seg_len"]
    n = nseg * seg
    src = torch.empty(n, dtype=torch.int32, device=dev)
    from paper_2503_05934_b200._lib import check
    check(L.ns_generate_i32(src.data_ptr(), n, 0, SEED, torch.cuda.current_stream().cuda_stream),
          "generate")
    w = src.clone()
    cfg = ns.find_config(g["config"])
    fn = lambda: ns.segmented_sort(w, seg, cfg, ns.Algorithm.quick_sort)  # noqa: E731
    restore = lambda: w.copy_(src)  # noqa: E731
    ms, how = device_ms(fn, restore, True, 5)
    restore()
    prof = _profile(L, fn)
    pre = w[: g["num_segments_checked"] * seg].cpu().numpy()
    v = w.view(nseg, seg)
    seg_sorted = bool((v[:, 1:] >= v[:, :-1]).all().item())
    ok = (_sha(pre) == g["output_prefix_sha256"] and seg_sorted and
          ns.multiset_digest(w) == ns.multiset_digest(src))
    res["segmented:3To5:65536x16384"] = {
        "workload": "BASELINE configs[3] segmented batch: 65,536 independent uniform-random "
                    "int32 arrays of 16,384 keys, quick sort 3To5 per segment",
        "n": n, "device_ms": ms, "timing": how, "gkeys_per_s": n / (ms * 1e-3) / 1e9,
        "model_bytes": 8 * n, "byte_model": "8n: one on-chip pass (read + write every key once)",
        "hbm_frac": 8 * n / (ms * 1e-3) / 1e9 / peak, "kernel_profile": prof,
        "verified": bool(ok),
        "verified_against": "SHA-256 of the reference's output on the first 1,024 segments "
                            "(golden.json) + every segment sorted + multiset digest"}
    del src, w, v
    ns.release_scratch()
    torch.cuda.empty_cache()
    return res


def attach_cpu(configs, cells):
    """Reference 1-core time per cell (same inputs) and the device speed-up."""
    if "cells" not in cells:
        return
    for name, rec in configs.items():
        key = name if name in cells["cells"] else name + ":1024"
        c = cells["cells"].get(key)
        if not c:
            continue
        cpu_ms = c["cpu_ms"]
        keys_gpu = rec.get("n") or rec.get("num_keys")
        if name.startswith("segmented"):  # 1,024 of the segments timed: per-key rate
            cpu_ms = cpu_ms * keys_gpu / c["keys_per_call"]
        rec["cpu_ref"] = {"ms": cpu_ms, "cores": 1, "kind": "reference",
                          "iterations": c["iterations"], "wall_ms": c["wall_ms"]}
        if c.get("note"):
            rec["cpu_ref"]["note"] = c["note"]
        rec["speedup_vs_ref_1core"] = cpu_ms / rec["device_ms"]
        if "e2e" in rec:
            rec["e2e"]["speedup_vs_ref_1core"] = cpu_ms / rec["e2e"]["ms"]


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
    """--extra: the §8(f) widenings — int64 keys (the reference's own benchmark
    type, full 64-bit values) and the stable key-value sort."""
    import numpy as np
    import torch
    peak = measured_peaks()[0]
    res = {}

    def single(name, algo, n):
        a = torch.from_numpy(ns.generate("random", n, SEED, dtype=np.int64)).to(dev)
        w = a.clone()
        cfg = ns.find_config("6To8" if algo == "merge" else "3To5")
        sort = ns.optimized_merge_sort if algo == "merge" else ns.optimized_quick_sort
        fn = lambda: sort(w, cfg)  # noqa: E731
        restore = lambda: w.copy_(a)  # noqa: E731
        ms, how = device_ms(fn, restore, algo == "merge" or QS_GRAPH_SAFE, 5)
        w.copy_(a)
        fn()
        rec = {"n": n, "device_ms": ms, "timing": how, "gkeys_per_s": n / (ms * 1e-3) / 1e9,
               "sorted": ns.count_inversions(w) == 0,
               "key": "int64 (the reference's own benchmark type, full 64-bit values)"}
        if algo == "merge" and n > (1 << 14):
            passes = 1 + max(0, (n - 1).bit_length() - 13)
            rec["hbm_frac_all_passes"] = 16 * n * passes / (ms * 1e-3) / 1e9 / peak
        res[name] = rec
        del a, w

    for n in (1_000_000, 1 << 28):
        single(f"ms_6to8_random_i64_{n}", "merge", n)
    for n in (1_000_000, 16_777_216):
        single(f"qs_3to5_random_i64_{n}", "quick", n)
    torch.cuda.empty_cache()
    n = 1 << 26
    kk = torch.from_numpy(ns.generate("random", n, SEED)).to(dev)
    vv = torch.arange(n, dtype=torch.int32, device=dev)
    wk, wv = kk.clone(), vv.clone()
    fn = lambda: ns.sort_pairs(wk, wv)  # noqa: E731
    restore = lambda: (wk.copy_(kk), wv.copy_(vv))  # noqa: E731
    ms, how = device_ms(fn, restore, True, 5)
    res["sort_pairs_i32_random_2^26"] = {"n": n, "device_ms": ms, "timing": how,
                                         "gkeys_per_s": n / (ms * 1e-3) / 1e9}
    del kk, vv, wk, wv
    torch.cuda.empty_cache()
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
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the per-config objects (BASELINE configs[0..3])")
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
