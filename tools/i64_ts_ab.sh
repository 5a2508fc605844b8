cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for v in build/variants/*.so; do
  echo "== $v"; cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  python -m pytest tests/test_gpu_int64.py -x -q -k "sizes or golden" 2>&1 | tail -1
  python tests/kind_profile.py merge 268435456 i64 | grep -E "call|tile"
done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
