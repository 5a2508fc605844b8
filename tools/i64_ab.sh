# int64 tile-sort variant A/B over prebuilt libraries (build/variants/*.so)
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  timeout 900 python -m pytest tests/test_gpu_int64.py -x -q 2>&1 | tail -1
  for n in 16777216 268435456; do python tests/kind_profile.py merge $n i64 | grep -E "call|tile|merge_pass"; done
  python tests/kind_profile.py quick 16777216 i64 | grep -E "call|bucket"
  python tests/size_sweep.py --i64 --min=20 --max=28 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
