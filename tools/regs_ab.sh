cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python tests/size_sweep.py --min=18 --max=30 | python -c "
import sys,json
print(' '.join(f\"{json.loads(l)['log2n']}:{json.loads(l)['ms']*1000:.1f}\" for l in sys.stdin))"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
