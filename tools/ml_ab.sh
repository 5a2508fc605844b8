cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  NSB_QS=2 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "quick or golden or adversarial" 2>&1 | tail -1
  python tests/kind_profile.py quick 67108864 | grep -E "call|count|scatter|bucket"
  python tests/size_sweep.py --quick --min=24 --max=28 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['ms']*1000,1), d['sorted'])"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
