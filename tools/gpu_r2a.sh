# round-2 parity additions + counters / memory / CLI on the GPU
timeout 1800 python -m pytest tests/test_gpu_parity_r2.py tests/test_gpu_loopback.py tests/test_gpu_memory.py tests/test_cli.py -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/r2a_tests.log 2>&1; echo "tests rc=$?"
tail -30 gpurun_out/r2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
