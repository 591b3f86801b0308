timeout 1200 python -m pytest tests/test_gpu_roe_split.py -q -x -p no:cacheprovider > gpurun_out/roe1_tests.log 2>&1; echo "roe tests rc=$?"
tail -30 gpurun_out/roe1_tests.log
timeout 600 python -m pytest tests/test_gpu_memory.py -q -x -p no:cacheprovider 2>&1 | tail -30
python tools/probe.py c4 --flux roe --tag roe_split > gpurun_out/roe1_probe.jsonl 2>&1
BF_ROE_SPLIT=0 python tools/probe.py c4 --flux roe --tag roe_ref >> gpurun_out/roe1_probe.jsonl 2>&1
python tools/probe.py c3 --tag c3_split >> gpurun_out/roe1_probe.jsonl 2>&1
BF_ROE_SPLIT=0 python tools/probe.py c3 --tag c3_ref >> gpurun_out/roe1_probe.jsonl 2>&1
cut -c1-420 gpurun_out/roe1_probe.jsonl
