cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python -m pytest tests/test_gpu_parity.py -x -q -k "batch or networks_exhaustive" 2>&1 | tail -1
  python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_2503_05934_b200 as ns
from oracle import oracle as O
offs, keys = O.generate_batch_i32(1 << 24, 42)
k = torch.from_numpy(keys).cuda(); o = torch.from_numpy(offs.view(np.int32)).cuda(); w = k.clone()
for _ in range(3): w.copy_(k); ns.sort_small_batch(w, o)
ts = []
for _ in range(10):
    w.copy_(k); a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); ns.sort_small_batch(w, o); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
nb = 8 * len(keys) + 4 * len(offs)
print('batch call ms', round(min(ts), 4), 'GB/s', round(nb / (min(ts) * 1e-3) / 1e9, 1))
PY
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
