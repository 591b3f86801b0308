: > gpurun_out/drift2.jsonl
for v in rcpn2 nofma; do
BFGPU_LIB=paper_2012_02925_b200/libbfgpu_$v.so python tools/drift_probe.py c1 250,1000,2000 >> gpurun_out/drift2.jsonl 2>>gpurun_out/drift2.err
done
cat gpurun_out/drift2.jsonl
timeout 600 ncu --set full --import-source on --clock-control none -k regex:roe_stage_kernel -c 2 -f -o gpurun_out/roe_v1 python tools/probe.py c4 --flux roe --steps 1 --warmup 0 > gpurun_out/ncu_roe.log 2>&1; echo "ncu rc=$?"
timeout 900 python -m pytest tests/test_gpu_memory.py "tests/test_gpu_parity_r2.py::test_c3_order_study_32_64_128_on_8_blocks" -q -p no:cacheprovider 2>&1 | tail -4
