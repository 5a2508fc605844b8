"""Debug helper (not collected): one small merge sort that takes the k-way path."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_05934_b200 as ns
from oracle import oracle as O
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
a = O.generate_i32("random", n, 42 + n)
t = torch.from_numpy(a).cuda()
try:
    ns.optimized_merge_sort(t, ns.find_config("6To8"))
except Exception as e:
    print("ERR", e)
torch.cuda.synchronize()
print("ok", np.array_equal(t.cpu().numpy(), np.sort(a)))
import ctypes as C
L = ns.lib()
if hasattr(L, "ns_debug_read"):
    buf = (C.c_int * 8)()
    L.ns_debug_read(buf)
    print("dbg", list(buf))
