# shared pairwise reciprocals in the Van Albada quotients: accuracy tests + A/B
timeout 1500 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_vl_split.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/ab_probe.sh c4 base nopair
