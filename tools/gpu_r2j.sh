# fused guard + fused fill heuristic: tests, then C1/C2/C4 timing A/B
timeout 1200 python -m pytest tests/test_gpu_fused_fill.py tests/test_gpu_graph.py tests/test_gpu_iterate_loop.py tests/test_gpu_vl_split.py -q -x -p no:cacheprovider 2>&1 | tail -5
: > gpurun_out/r2j_probe.jsonl
for c in c1 c2 c4; do
  BF_FUSED_GUARD=0 BF_FUSED_FILL=0 timeout 300 python tools/probe.py $c --tag "${c}_sep" >> gpurun_out/r2j_probe.jsonl 2>&1
  timeout 300 python tools/probe.py $c --tag "${c}_default" >> gpurun_out/r2j_probe.jsonl 2>&1
done
BF_FUSED_FILL=1 timeout 300 python tools/probe.py c1 --tag "c1_fill1" >> gpurun_out/r2j_probe.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2j_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'noprof', round(d['ms_per_step_noprof'],4), 'mcups_noprof', round(d['mcups_noprof']), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4))
"
