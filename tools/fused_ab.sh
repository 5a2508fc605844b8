# in-kernel split search (FUSED) threshold A/B: merge sort time per n
for f in 0 512 1024 2048 4096 16384; do
  NSB_FUSED_MAX=$f python tests/size_sweep.py --min=20 --max=26 | python -c "
import sys,json
print('fused_max=$f', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
