"""Small fixed workload for ncu captures (not collected by pytest).

    python tests/prof_run.py merge 268435456     # one warm-up sort + one sort
    python tests/prof_run.py batch 16777216
    python tests/prof_run.py segmented 65536
    python tests/prof_run.py quick 16777216
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "merge"
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 28
    dev = torch.device("cuda:0")
    L = ns.lib()
    s = torch.cuda.current_stream().cuda_stream
    if mode == "batch":
        from oracle import oracle as O
        offs, keys = O.generate_batch_i32(n, 42)
        k = torch.from_numpy(keys).to(dev)
        o = torch.from_numpy(offs.view("int32")).to(dev)
        for _ in range(2):
            w = k.clone()
            ns.sort_small_batch(w, o)
    elif mode == "segmented":
        seg = 16384
        a = torch.empty(n * seg, dtype=torch.int32, device=dev)
        check(L.ns_generate_i32(a.data_ptr(), a.numel(), 0, 42, s), "gen")
        for _ in range(2):
            w = a.clone()
            ns.segmented_sort(w, seg, ns.find_config("3To5"), ns.Algorithm.quick_sort)
    else:
        a = torch.empty(n, dtype=torch.int32, device=dev)
        check(L.ns_generate_i32(a.data_ptr(), n, 0, 42, s), "gen")
        fn = ns.optimized_merge_sort if mode == "merge" else ns.optimized_quick_sort
        cfg = ns.find_config("6To8" if mode == "merge" else "3To5")
        for _ in range(2):
            w = a.clone()
            fn(w, cfg)
        assert ns.count_inversions(w) == 0
    torch.cuda.synchronize()
    print("prof_run ok", mode, n)


if __name__ == "__main__":
    main()
