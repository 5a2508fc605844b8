cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python -m pytest tests/test_gpu_parity.py -x -q -k "quick or golden" 2>&1 | tail -1
  python tests/kind_profile.py quick 16777216 | grep -E "call|count|scatter|bucket"
  python tests/size_sweep.py --quick --min=20 --max=25 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['ms']*1000,1), d['sorted'])"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
