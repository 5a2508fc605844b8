# partition with block samples (NSB_SAMPLES=1, default) vs the plain search
python -m pytest tests/test_gpu_parity.py tests/test_gpu_int64.py -x -q -k "sizes or golden or every_config or duplicates or kway or full_size or beyond" 2>&1 | tail -1
for v in 0 1; do echo "== NSB_SAMPLES=$v"; NSB_SAMPLES=$v python tests/kind_profile.py merge 1073741824 | grep -E "partition|merge_pass"; NSB_SAMPLES=$v python tests/size_sweep.py --min=24 --max=30; done
