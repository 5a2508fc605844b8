"""Builder tool: quick sort vs merge sort device time by CUDA-graph replay."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_05934_b200 as ns  # noqa: E402

bench.QS_GRAPH_SAFE = True
dev = torch.device("cuda:0")
for lg in range(14, 24):
    for n in ((1 << lg), (1 << lg) + (1 << (lg - 1))):
        a = torch.from_numpy(ns.generate("random", n, 42)).to(dev)
        row = [f"{n:>9d}"]
        for fn, cfgn in ((ns.optimized_merge_sort, "6To8"), (ns.optimized_quick_sort, "3To5")):
            w = a.clone()
            cfg = ns.find_config(cfgn)
            ms, _ = bench.device_ms(lambda: fn(w, cfg), lambda: w.copy_(a), True, 20)
            row.append(f"{ms*1000:8.1f} us")
        print("  ".join(row))
