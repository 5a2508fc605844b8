# A/B of prebuilt library variants (build/variants/*.so): parity subset,
# tile-sort / merge-pass split at 2^28 and 2^30, segmented 65,536 x 16,384,
# merge-sort size sweep.  Usage: bash tools/ab_all.sh [pytest -k expr]
K=${1:-"segmented or sizes or distributions"}
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"
  cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "$K" 2>&1 | tail -1
  for n in 268435456 1073741824; do
    python tests/kind_profile.py merge $n | grep -E "call|merge_pass|tile"
  done
  python tools/seg_time.py
  python tests/size_sweep.py --min=${MINLG:-20} --max=30 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['ms']*1000,1), d['sorted'])"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
