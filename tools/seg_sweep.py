import sys, torch
sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns
from paper_2503_05934_b200._lib import check
L = ns.lib()
total = 1 << 26
a = torch.empty(total, dtype=torch.int32, device='cuda')
check(L.ns_generate_i32(a.data_ptr(), total, 0, 42, torch.cuda.current_stream().cuda_stream), 'g')
for algo, cfgn in ((ns.Algorithm.merge_sort, '6To8'), (ns.Algorithm.quick_sort, '3To5')):
    cfg = ns.find_config(cfgn)
    for seg in (8, 16, 32, 64, 128, 256, 512, 1000, 2048, 4096, 5000, 8192, 12000, 16384, 16385, 20000, 32768, 50000, 65536, 100000, 262144, 1 << 20, 1 << 22):
        nseg = total // seg
        n = nseg * seg
        w = a[:n].clone()
        ts = []
        for it in range(4):
            w.copy_(a[:n])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ns.segmented_sort(w, seg, cfg, algo)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        v = w.view(nseg, seg)
        ok = bool((v[:, 1:] >= v[:, :-1]).all()) if seg > 1 else True
        print(algo.name, seg, nseg, round(min(ts), 3), 'ms', round(min(ts) * 1e6 / n, 2), 'ns/Kkey' if False else 'ps/key x1e3', ok)
