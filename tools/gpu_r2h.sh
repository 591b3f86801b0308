timeout 900 python -m pytest tests/test_gpu_iterate_loop.py tests/test_gpu_graph.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/r2h_probe.jsonl
for c in c1 c2 c3 c4; do python tools/probe.py $c --tag "$c" >> gpurun_out/r2h_probe.jsonl 2>&1; done
python tools/probe.py c1 --flux roe --tag c1_roe >> gpurun_out/r2h_probe.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2h_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'noprof', round(d['ms_per_step_noprof'],4), 'mcups_noprof', round(d['mcups_noprof']), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4))
"
