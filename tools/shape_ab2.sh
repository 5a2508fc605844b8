for v in 0 14 13 16; do
  NSB_V2=$v python tests/size_sweep.py --min=24 --max=30 | python -c "
import sys,json
print('v2=$v', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
