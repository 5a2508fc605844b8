cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python tests/kind_profile.py merge 268435456 i64 | grep -E "call|tile"
  python tests/kind_profile.py quick 16777216 i64 | grep -E "call|bucket"
  python tests/kind_profile.py quick 16777216 | grep -E "call|bucket"
  python tools/seg_time.py
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
