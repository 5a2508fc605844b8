"""Per-kernel-class device times of one sort (library profiler), for tuning
runs under different NSB_* environment knobs.  Not collected by pytest.

    NSB_TILE=16384 python tests/tune_run.py merge 268435456
"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "merge"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    dev = torch.device("cuda:0")
    L = ns.lib()
    s = torch.cuda.current_stream().cuda_stream
    if mode == "batch":
        from oracle import oracle as O
        offs, keys = O.generate_batch_i32(n, 42)
        a = torch.from_numpy(keys).to(dev)
        o = torch.from_numpy(offs.view("int32")).to(dev)
    else:
        a = torch.empty(n, dtype=torch.int32, device=dev)
        check(L.ns_generate_i32(a.data_ptr(), n, 0, 42, s), "gen")
    w = a.clone()
    if mode == "batch":
        fn = lambda: ns.sort_small_batch(w, o)  # noqa: E731
    elif mode == "merge":
        fn = lambda: ns.optimized_merge_sort(w, ns.find_config("6To8"))  # noqa: E731
    elif mode == "quick":
        fn = lambda: ns.optimized_quick_sort(w, ns.find_config("3To5"))  # noqa: E731
    elif mode == "segmented":
        fn = lambda: ns.segmented_sort(w, 16384, ns.find_config("3To5"))  # noqa: E731
    fn()
    res = {"mode": mode, "n": n, "env": {k: v for k, v in os.environ.items() if k.startswith("NSB_")}}
    tot = []
    for _ in range(reps):
        w.copy_(a)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        tot.append(e0.elapsed_time(e1))
    res["ms"] = min(tot)
    res["gkeys_s"] = n / (res["ms"] * 1e-3) / 1e9
    w.copy_(a)
    torch.cuda.synchronize()
    check(L.ns_profile_enable(1), "p")
    fn()
    torch.cuda.synchronize()
    prof = {}
    for k in range(L.ns_profile_kinds()):
        t, c = C.c_double(), C.c_uint64()
        check(L.ns_profile_read(k, C.byref(t), C.byref(c)), "r")
        if c.value:
            prof[L.ns_profile_kind_name(k).decode()] = [round(t.value, 4), c.value,
                                                        round(t.value / c.value, 4)]
    L.ns_profile_enable(0)
    res["prof_ms_launches_avg"] = prof
    if mode not in ("segmented", "batch"):
        assert ns.count_inversions(w) == 0
    print(json.dumps(res))


if __name__ == "__main__":
    main()
