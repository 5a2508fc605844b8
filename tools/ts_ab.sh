cp paper_2503_05934_b200/lib/libnetsort_b200.so /tmp/lib_orig.so
for rep in 1 2; do
for v in build/variants/*.so; do
  cp "$v" paper_2503_05934_b200/lib/libnetsort_b200.so
  echo "$v $(python tests/kind_profile.py merge 1073741824 | grep tile_sort) $(python tools/seg_time.py)"
done; done
cp /tmp/lib_orig.so paper_2503_05934_b200/lib/libnetsort_b200.so
