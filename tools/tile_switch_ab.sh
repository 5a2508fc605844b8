for t in 0 8192 16384; do
  if [ $t = 0 ]; then unset NSB_TILE; else export NSB_TILE=$t; fi
  python tests/size_sweep.py --min=19 --max=25 | python -c "
import sys,json
print('tile=$t', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
