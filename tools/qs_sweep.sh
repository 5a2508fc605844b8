# quick sort: single-level (NSB_QS=1) vs multi-level (NSB_QS=2) partition
for m in 1 2; do echo "== NSB_QS=$m"; NSB_QS=$m python tests/size_sweep.py --quick --min=15 --max=28; done
