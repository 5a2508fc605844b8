"""Debug helper: run the device sorts size by size, synchronising after each
call, and report the first failing case.  Not collected by pytest.

    python tests/debug_sizes.py [merge|quick|host|batch] [sizes...]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05934_b200 as ns  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "merge"
    sizes = [int(x) for x in sys.argv[2:]] or [
        2, 3, 8, 9, 31, 32, 33, 255, 256, 257, 1000, 4096, 8191, 8192, 8193, 16383, 16384, 16385,
        20000, 32768, 65537, 100000, 1000000]
    dev = torch.device("cuda:0")
    for n in sizes:
        print(f"{mode} n={n} ...", flush=True)
        a = O.generate_i32("random", n, 42 + n)
        if mode == "host":
            h = a.copy()
            ns.optimized_merge_sort(h, ns.find_config("6To8"))
            ok = np.array_equal(h, np.sort(a))
        else:
            t = torch.from_numpy(a).to(dev)
            fn = ns.optimized_merge_sort if mode == "merge" else ns.optimized_quick_sort
            fn(t, ns.find_config("6To8" if mode == "merge" else "3To5"))
            torch.cuda.synchronize()
            ok = np.array_equal(t.cpu().numpy(), np.sort(a))
        print(f"   ok={ok}", flush=True)
        if not ok:
            break


if __name__ == "__main__":
    main()
