# int64 merge-sort tile A/B: NSB_TILE64=2 (<512,16>, 8192 keys) vs 3 (<1024,16>, 16384 keys from 2^21)
for v in 2 3; do
  export NSB_TILE64=$v; echo "== NSB_TILE64=$v"
  timeout 900 python -m pytest tests/test_gpu_int64.py -x -q 2>&1 | tail -1
  python tests/kind_profile.py merge 268435456 i64 | grep -E "call|tile|merge_pass"
  python tests/size_sweep.py --i64 --min=20 --max=28 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
unset NSB_TILE64
echo "== int32 sweep (fused threshold by tile size)"
python tests/size_sweep.py --min=20 --max=26 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
