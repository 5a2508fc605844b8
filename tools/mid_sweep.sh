# merge-pass tile shapes across sizes (env knobs of netsort_capi.cu MergeTuning)
for cfg in "NSB_V2=0" "NSB_V2=3" "NSB_V2=5" "NSB_V2=6" "NSB_V2=9" "NSB_V2=11"; do
  echo "== $cfg"
  env $cfg python tests/size_sweep.py --min=16 --max=30
done
