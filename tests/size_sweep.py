"""Merge-sort throughput across sizes (not collected by pytest).

    python tests/size_sweep.py [--i64] [--quick]

For each n, the sort is captured in a CUDA graph together with an input
restore (D2D copy) and replayed; the restore-only graph is timed separately
and subtracted.  Prints one JSON line per size with Gkeys/s and the byte-model
fraction (8 B/key per pass for int32, 16 for int64; passes = 1 tile pass +
one per doubling above the tile: 16384 int32 keys from 2^21 keys up, else
8192) of the measured HBM bandwidth.
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402


def timed_graph(fn, restore, reps):
    for _ in range(3):
        restore()
        fn()
    torch.cuda.synchronize()
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
    return out[0] - out[1]


def main():
    i64 = "--i64" in sys.argv
    quick = "--quick" in sys.argv
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        peak = float(json.load(f)["hbm_gbs"])
    dev = torch.device("cuda:0")
    L = ns.lib()
    kb = 8 if i64 else 4
    top = 29 if i64 else 30
    lo = 14
    for a in sys.argv[1:]:
        if a.startswith("--max="):
            top = int(a[6:])
        if a.startswith("--min="):
            lo = int(a[6:])
    for lg in range(lo, top + 1):
        n = 1 << lg
        src = torch.empty(n, dtype=torch.int32, device=dev)
        check(L.ns_generate_i32(src.data_ptr(), n, 0, 42, torch.cuda.current_stream().cuda_stream),
              "gen")
        if i64:
            src = (src.to(torch.int64) << 32) | src.to(torch.int64)
        w = src.clone()
        cfg = ns.find_config("3To5" if quick else "6To8")
        fn = (lambda: ns.optimized_quick_sort(w, cfg)) if quick else \
            (lambda: ns.optimized_merge_sort(w, cfg))
        restore = lambda: w.copy_(src)  # noqa: E731
        reps = max(3, min(200, (1 << 26) // n))
        if quick:  # host round trips: time per call with events
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
            ms = sorted(ts)[len(ts) // 2]
        else:
            ms = timed_graph(fn, restore, reps)
        restore()
        fn()
        # the library's tile: 16384 int32 keys from 2^21 up, else 8192
        tile_lg = 14 if (kb == 4 and lg >= 21) else 13
        passes = 1 + max(0, lg - tile_lg)
        rec = {"n": n, "log2n": lg, "key_bytes": kb, "algo": "quick" if quick else "merge",
               "ms": ms, "gkeys_per_s": n / (ms * 1e-3) / 1e9,
               "frac_all_passes": kb * 2 * n * passes / (ms * 1e-3) / 1e9 / peak,
               "frac_single_pass": kb * 2 * n / (ms * 1e-3) / 1e9 / peak,
               "sorted": ns.count_inversions(w) == 0}
        print(json.dumps(rec), flush=True)
        del src, w
        ns.release_scratch()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
