"""Merge-sort device time (CUDA-graph replay, input restore subtracted) for
small n, 6To8 random int32: python tools/small_sweep.py [n ...]"""
import os
import sys

import torch

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402
from size_sweep import timed_graph  # noqa: E402

L = ns.lib()
sizes = [int(a) for a in sys.argv[1:]] or [2000, 4096, 6000, 8192, 10000, 12000, 16384, 25000,
                                          32768, 65536, 100000]
cfg = ns.find_config("6To8")
out = []
for n in sizes:
    src = torch.empty(n, dtype=torch.int32, device='cuda')
    check(L.ns_generate_i32(src.data_ptr(), n, 0, 42, torch.cuda.current_stream().cuda_stream), "g")
    w = src.clone()
    ms = timed_graph(lambda: ns.optimized_merge_sort(w, cfg), lambda: w.copy_(src), 200)
    w.copy_(src)
    ns.optimized_merge_sort(w, cfg)
    ok = bool(torch.equal(w, torch.sort(src).values))
    out.append(f"{n}:{ms * 1e3:.1f}{'' if ok else '!BAD'}")
print(os.environ.get("TAG", ""), " ".join(out))
