python tools/drift_probe.py c1 250,1000,2000 > gpurun_out/drift.jsonl 2>gpurun_out/drift.err
BFGPU_LIB=paper_2012_02925_b200/libbfgpu_rcpfull.so python tools/drift_probe.py c1 250,1000,2000 >> gpurun_out/drift.jsonl 2>>gpurun_out/drift.err
cat gpurun_out/drift.jsonl
python tools/probe.py c4 --tag base > gpurun_out/r2b_probe.jsonl 2>>gpurun_out/drift.err
BFGPU_LIB=paper_2012_02925_b200/libbfgpu_rcpfull.so python tools/probe.py c4 --tag rcpfull >> gpurun_out/r2b_probe.jsonl 2>>gpurun_out/drift.err
python tools/probe.py c4 --tag base2 >> gpurun_out/r2b_probe.jsonl 2>>gpurun_out/drift.err
BFGPU_LIB=paper_2012_02925_b200/libbfgpu_rcpfull.so python tools/probe.py c4 --tag rcpfull2 >> gpurun_out/r2b_probe.jsonl 2>>gpurun_out/drift.err
cut -c1-400 gpurun_out/r2b_probe.jsonl
timeout 900 python -m pytest tests/test_gpu_memory.py "tests/test_gpu_parity_r2.py::test_c3_order_study_32_64_128_on_8_blocks" -q -p no:cacheprovider 2>&1 | tail -5
