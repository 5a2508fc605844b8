"""Builder tool: both sorts at n keys over input shapes that stress pivot
selection and duplicates (device time, best of 5, checked against torch.sort)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
DT = torch.int64 if len(sys.argv) > 2 and sys.argv[2] == 'i64' else torch.int32
dev = torch.device('cuda')
g = torch.Generator(device='cuda').manual_seed(1)
r = torch.randint(0, 2**31 - 1, (n,), device=dev, dtype=DT, generator=g)
ar = torch.arange(n, device=dev, dtype=DT)
shapes = {
    'random': r,
    'sorted': ar,
    'reversed': ar.flip(0).contiguous(),
    'all_equal': torch.full((n,), 7, device=dev, dtype=DT),
    'two_values': (r & 1),
    '16_values': (r & 15),
    '1000_values': (r % 1000),
    'organ_pipe': torch.minimum(ar, ar.flip(0)).contiguous(),
    'sawtooth_1024': (ar & 1023),
    'mostly_equal_1pct_random': torch.where((r % 100) == 0, r, torch.full_like(r, 123456)),
    'int_extremes': torch.where((r & 1) == 0, torch.full_like(r, -2**31), torch.full_like(r, 2**31 - 1)),
    'negative_random': (r - 2**30),
}
for name, a in shapes.items():
    want = torch.sort(a).values
    for algo, cfgn, fn in (('merge', '6To8', ns.optimized_merge_sort), ('quick', '3To5', ns.optimized_quick_sort)):
        cfg = ns.find_config(cfgn)
        w = a.clone()
        ts = []
        for _ in range(5):
            w.copy_(a)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(w, cfg)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        print(f'{name:28s} {algo:6s} {min(ts)*1000:9.1f} us  ok={bool(torch.equal(w, want))}')
