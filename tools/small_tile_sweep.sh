# merge-sort time (us) per forced tile size (NSB_TILE) for n = 2^14..2^22 (graph replay)
for t in 0 1024 2048 4096 8192 16384; do
  echo "== NSB_TILE=$t"
  if [ $t = 0 ]; then unset NSB_TILE; else export NSB_TILE=$t; fi
  python tests/size_sweep.py --min=14 --max=22 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
