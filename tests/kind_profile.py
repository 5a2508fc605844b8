"""Per-kernel-class device time of one sort from the library's own launch
events (ns_profile_*), not under a profiler (not collected by pytest).

    python tests/kind_profile.py quick 16777216 [i64]
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "quick"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
    L = ns.lib()
    dev = torch.device("cuda:0")
    src = torch.empty(n, dtype=torch.int32, device=dev)
    check(L.ns_generate_i32(src.data_ptr(), n, 0, 42, torch.cuda.current_stream().cuda_stream), "gen")
    if len(sys.argv) > 3 and sys.argv[3] == "i64":
        src = (src.to(torch.int64) << 32) | src.to(torch.int64)
    fn = ns.optimized_quick_sort if mode == "quick" else ns.optimized_merge_sort
    cfg = ns.find_config("3To5" if mode == "quick" else "6To8")
    for rep in range(4):
        w = src.clone()
        torch.cuda.synchronize()
        if rep == 3:
            check(L.ns_profile_enable(1), "prof")
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(w, cfg)
        b.record()
        torch.cuda.synchronize()
    total = a.elapsed_time(b)
    print(f"{mode} n={n}: call {total * 1e3:.1f} us")
    for k in range(L.ns_profile_kinds()):
        t, c = C.c_double(), C.c_uint64()
        check(L.ns_profile_read(k, C.byref(t), C.byref(c)), "read")
        if c.value:
            print(f"  {L.ns_profile_kind_name(k).decode():18s} {t.value * 1e3:9.1f} us  {c.value} launches")
    check(L.ns_profile_enable(0), "prof")


if __name__ == "__main__":
    main()
