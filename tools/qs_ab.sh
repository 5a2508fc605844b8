# quick-sort variant A/B over prebuilt libraries (build/variants/*.so)
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "quick or adversarial or segmented or i64" 2>&1 | tail -1
  python tests/size_sweep.py --quick --min=20 --max=27 | python -c "
import sys,json
print('quick', ' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
  python tests/kind_profile.py quick 16777216 | grep -E "call|sample|tile|merge|bucket"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
