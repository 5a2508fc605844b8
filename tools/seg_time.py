"""Segmented 65,536 x 16,384 random int32 (BASELINE config 4's batch), best of 5 (device time)."""
import sys

import torch

sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402

L = ns.lib()
n = 65536 * 16384
a = torch.empty(n, dtype=torch.int32, device='cuda')
check(L.ns_generate_i32(a.data_ptr(), n, 0, 42, torch.cuda.current_stream().cuda_stream), 'g')
cfg = ns.find_config('3To5')
w = a.clone()
for _ in range(2):
    w.copy_(a)
    ns.segmented_sort(w, 16384, cfg, ns.Algorithm.quick_sort)
ts = []
for _ in range(5):
    w.copy_(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ns.segmented_sort(w, 16384, cfg, ns.Algorithm.quick_sort)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print('segmented ms', round(min(ts), 3))
