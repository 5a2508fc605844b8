# int64 merge-pass tile shapes (NSB_V2_64, netsort_capi.cu)
for v in 0 1 2 3; do echo "== NSB_V2_64=$v"; NSB_V2_64=$v python tests/size_sweep.py --i64 --min=18 --max=29; done
