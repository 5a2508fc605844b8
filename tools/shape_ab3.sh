for v in -1 15; do
  NSB_V2=$v python tests/size_sweep.py --min=24 --max=30 | python -c "
import sys,json
print('v2=$v', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
  NSB_V2=$v python tests/kind_profile.py merge 1073741824 | grep -E "partition|merge_pass"
done
