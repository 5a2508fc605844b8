"""Quick-sort timing probe (builder tool): device time by CUDA-graph replay and
the per-kernel split from the library's launch events, checked sorted."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_05934_b200 as ns  # noqa: E402

bench.QS_GRAPH_SAFE = True
L = ns.lib()
dev = torch.device("cuda:0")
out = {}
sizes = [int(x) for x in (sys.argv[1:] or ["1000000", "16777216"])]
for n in sizes:
    for dist in ("random", "sorted"):
        a = torch.from_numpy(ns.generate(dist, n, 42)).to(dev)
        w = a.clone()
        cfg = ns.find_config("3To5")
        fn = lambda: ns.optimized_quick_sort(w, cfg)  # noqa: E731
        restore = lambda: w.copy_(a)  # noqa: E731
        ms, how = bench.device_ms(fn, restore, True, 20)
        restore()
        prof = bench._profile(L, fn)
        ok = ns.count_inversions(w) == 0 and ns.multiset_digest(w) == ns.multiset_digest(a)
        out[f"{dist}:{n}"] = {"ms": ms, "ok": ok,
                              "prof": {k: (round(v["ms"], 4), v["launches"]) for k, v in prof.items()}}
        print(dist, n, round(ms * 1e3, 1), "us", ok, out[f"{dist}:{n}"]["prof"], flush=True)
print(json.dumps(out))
