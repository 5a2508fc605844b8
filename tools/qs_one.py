"""One quick sort (builder tool, for ncu captures): n keys, distribution."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2503_05934_b200 as ns  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
dist = sys.argv[2] if len(sys.argv) > 2 else "random"
a = torch.from_numpy(ns.generate(dist, n, 42)).to("cuda:0")
w = a.clone()
cfg = ns.find_config("3To5")
for _ in range(2):
    w.copy_(a)
    ns.optimized_quick_sort(w, cfg)
torch.cuda.synchronize()
assert ns.count_inversions(w) == 0
print("ok")
