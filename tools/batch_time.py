"""Base-case batch (BASELINE config 2: 2^24 ragged int32 arrays, lengths 3..8):
kernel time from the library's own launch events, median of 7 runs."""
import ctypes as C
import statistics
import sys

import torch

sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns  # noqa: E402
from paper_2503_05934_b200._lib import check  # noqa: E402
from oracle import oracle as O  # noqa: E402  (checker)

L = ns.lib()
offs, keys = O.generate_batch_i32(1 << 24, 42)
k = torch.from_numpy(keys).cuda()
o = torch.from_numpy(offs.view("int32")).cuda()
w = k.clone()
ns.sort_small_batch(w, o)
ok = bool(torch.equal(w.cpu(), torch.from_numpy(O.sort_small_batch(keys, offs))))
ts = []
for _ in range(7):
    w.copy_(k)
    torch.cuda.synchronize()
    check(L.ns_profile_enable(1), "p")
    ns.sort_small_batch(w, o)
    torch.cuda.synchronize()
    tot = 0.0
    for kk in range(L.ns_profile_kinds()):
        t, c = C.c_double(), C.c_uint64()
        check(L.ns_profile_read(kk, C.byref(t), C.byref(c)), "r")
        tot += t.value
    check(L.ns_profile_enable(0), "p")
    ts.append(tot)
ms = statistics.median(ts)
nbytes = 8 * len(keys) + 4 * len(offs)
print(f"batch kernel {ms * 1e3:.1f} us  {nbytes / ms / 1e6:.0f} GB/s  parity={ok}")
