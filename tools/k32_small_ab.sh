# tile shape at small n: NSB_K32=1 (<256,32> 8192-key tiles) vs 0 (<512,16>)
for v in 1 0; do
  NSB_K32=$v python tools/small_sweep.py 10000 25000 65536 100000 262144 524288 1000000 2097152 4194304 | sed "s/^/K32=$v /"
done
