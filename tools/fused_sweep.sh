# in-kernel (fused) split search vs the sample-bracketed partition kernel, by pass size
for f in 0 1024 4096; do echo "== NSB_FUSED_MAX=$f"; NSB_FUSED_MAX=$f python tests/size_sweep.py --min=20 --max=27; done
