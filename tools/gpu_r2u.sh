# vec2 COPY items: parity subset, then C4 / C2 ghost A/B
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fused_fill.py tests/test_gpu_vl_split.py tests/test_gpu_golden.py tests/test_gpu_loopback.py -q -x -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/vec2.jsonl
for rep in 1 2; do for c in c4 c2; do
  BF_GHOST_VEC2=0 timeout 300 python tools/probe.py $c --tag "${c}_scalar" >> gpurun_out/vec2.jsonl 2>&1
  timeout 300 python tools/probe.py $c --tag "${c}_vec2" >> gpurun_out/vec2.jsonl 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/vec2.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4))
"
