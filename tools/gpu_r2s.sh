# persistent segments: parity tests, then C4 and box:128 A/B (prev build / tiles / segments)
timeout 900 python -m pytest tests/test_gpu_vl_split.py tests/test_gpu_iterate_loop.py tests/test_gpu_graph.py tests/test_gpu_parity_r2.py tests/test_gpu_fused_fill.py -q -x -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/seg.jsonl
for rep in 1 2; do
for c in c4 box:128; do
  BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_prev.so timeout 300 python tools/probe.py $c --tag "${c}_prev" >> gpurun_out/seg.jsonl 2>&1
  BF_SEGMENTS=0 timeout 300 python tools/probe.py $c --tag "${c}_tiles" >> gpurun_out/seg.jsonl 2>&1
  timeout 300 python tools/probe.py $c --tag "${c}_segs" >> gpurun_out/seg.jsonl 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/seg.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'frac', round(d['stage_hbm_frac'],4))
"
