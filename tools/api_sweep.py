"""Builder tool: device time of the other entry points over sizes around their
internal thresholds (best of 4; every result checked), to spot cliffs."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns  # noqa: E402

dev = torch.device('cuda')
g = torch.Generator(device='cuda').manual_seed(1)


def timed(fn, restore, reps=4):
    best = 1e9
    for _ in range(reps):
        restore()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def rnd(n, dt=torch.int32):
    return torch.randint(0, 2**31 - 1, (n,), device=dev, dtype=dt, generator=g)


print('== quick / merge sort around the tile and level thresholds (int32)')
for n in (16384, 16385, 20000, 32768, 40000, 65536, 100000, 300000, (1 << 21) - 1, (1 << 21) + 1,
          3_000_000, (1 << 23) + 1, (1 << 27), (1 << 28)):
    a = rnd(n)
    want = torch.sort(a).values
    row = [f'{n:>10d}']
    for fn, cfgn in ((ns.optimized_merge_sort, '6To8'), (ns.optimized_quick_sort, '3To5')):
        w = a.clone()
        cfg = ns.find_config(cfgn)
        t = timed(lambda: fn(w, cfg), lambda: w.copy_(a))
        row.append(f'{t*1000:9.1f} us {n/t/1e6:7.2f} Gk/s ok={bool(torch.equal(w, want))}')
    print('  '.join(row))

print('== sort_pairs / argsort (int32 keys, 4-byte payload)')
for n in (10_000, 1 << 20, 1 << 24, 1 << 27):
    k = rnd(n)
    v = torch.arange(n, device=dev, dtype=torch.int32)
    kk, vv = k.clone(), v.clone()
    t = timed(lambda: ns.sort_pairs(kk, vv), lambda: (kk.copy_(k), vv.copy_(v)))
    ok = bool(torch.equal(kk, torch.sort(k, stable=True).values)) and bool(torch.equal(k[vv.long()], kk))
    kk.copy_(k)
    t2 = timed(lambda: ns.argsort(kk), lambda: kk.copy_(k))
    print(f'{n:>10d}  pairs {t*1000:9.1f} us {n/t/1e6:6.2f} Gk/s ok={ok}   argsort {t2*1000:9.1f} us')

print('== merge(a, left, mid, right): two sorted runs, skewed splits')
n = 1 << 24
base = torch.sort(rnd(n)).values
for frac in (0.5, 0.01, 0.99, 1e-6):
    nl = max(1, int(n * frac))
    a = torch.cat([torch.sort(rnd(nl)).values, torch.sort(rnd(n - nl)).values])
    w = a.clone()
    t = timed(lambda: ns.merge(w, 0, nl - 1, n - 1), lambda: w.copy_(a))
    print(f'  n_left={nl:>9d}  {t*1000:8.1f} us ok={bool(torch.equal(w, torch.sort(a).values))}')

print('== sort_small_batch: 2^22 arrays by length distribution')
na = 1 << 22
for name, lens in (('uniform 3..8', np.random.default_rng(1).integers(3, 9, na)),
                   ('all 8', np.full(na, 8)), ('all 3', np.full(na, 3)), ('all 1', np.full(na, 1)),
                   ('0..8', np.random.default_rng(2).integers(0, 9, na)),
                   ('sorted lengths', np.sort(np.random.default_rng(3).integers(0, 9, na)))):
    offs = np.zeros(na + 1, dtype=np.uint32)
    offs[1:] = np.cumsum(lens)
    nk = int(offs[-1])
    k = rnd(nk)
    o = torch.from_numpy(offs.view(np.int32)).to(dev)
    w = k.clone()
    t = timed(lambda: ns.sort_small_batch(w, o), lambda: w.copy_(k))
    print(f'  {name:16s} keys={nk:>9d}  {t*1000:8.1f} us  {nk/t/1e6:7.1f} Gk/s')
