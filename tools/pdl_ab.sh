# programmatic dependent launch on / off
python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "sizes or golden or every_config or duplicates or segmented or merge" 2>&1 | tail -1
for v in 0 2; do echo "== NSB_PDL=$v"; NSB_PDL=$v python tests/size_sweep.py --min=14 --max=30; done
