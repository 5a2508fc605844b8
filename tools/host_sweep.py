"""Builder tool: the host-array entry points (pageable numpy in place) over
sizes around their internal thresholds: wall time per call, checked."""
import sys
import time

import numpy as np

sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns  # noqa: E402

rng = np.random.default_rng(1)
for dt in (np.int32, np.int64):
    for n in (100, 8192, 8193, 16384, 16385, 100_000, 1 << 20, (1 << 22) - 1, 1 << 22, (1 << 23) - 1,
              1 << 23, (1 << 23) + 1, 1 << 24, 1 << 26):
        a = rng.integers(0, 2**31 - 1, n).astype(dt)
        want = np.sort(a)
        row = [f'{np.dtype(dt).name} {n:>9d}']
        for fn, cfgn in ((ns.optimized_merge_sort, '6To8'), (ns.optimized_quick_sort, '3To5')):
            cfg = ns.find_config(cfgn)
            best = 1e9
            for _ in range(4):
                w = a.copy()
                t0 = time.perf_counter()
                fn(w, cfg)
                best = min(best, time.perf_counter() - t0)
            row.append(f'{best*1e6:10.1f} us {n/best/1e9:6.3f} Gk/s ok={bool(np.array_equal(w, want))}')
        print('  '.join(row))
