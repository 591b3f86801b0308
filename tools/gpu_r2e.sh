timeout 1200 python -m pytest tests/test_gpu_roe_split.py tests/test_gpu_memory.py tests/test_gpu_parity_r2.py -q -x -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2e_tests.log
python tools/probe.py c4 --flux roe --tag roe_v2 > gpurun_out/r2e_probe.jsonl 2>&1
python tools/probe.py c3 --tag c3_v2 >> gpurun_out/r2e_probe.jsonl 2>&1
python tools/probe.py c4 --tag vl_rcpfull >> gpurun_out/r2e_probe.jsonl 2>&1
cut -c1-300 gpurun_out/r2e_probe.jsonl
python tools/drift_probe.py c1 250,1000,2000 > gpurun_out/drift3.jsonl 2>&1; cat gpurun_out/drift3.jsonl
