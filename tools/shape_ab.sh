# merge-pass tile shape per size (NSB_V2 forces one shape for every pass)
for v in -1 0 12 13 14 6 15 16; do
  NSB_V2=$v python tests/size_sweep.py --min=20 --max=27 | python -c "
import sys,json
print('v2=$v', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
