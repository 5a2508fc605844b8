# A/B of prebuilt library variants (build/variants/*.so) on the same box
cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"
  cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python tests/kind_profile.py merge 268435456 | grep -E "merge_pass|tile"
  python tests/size_sweep.py --min=${MINLG:-24} --max=30 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['log2n'], round(d['ms']*1000,1), d['sorted'])"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
