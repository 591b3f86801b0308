# guard with early RunState loads: iterate-loop tests, C1 timing
timeout 900 python -m pytest tests/test_gpu_iterate_loop.py tests/test_gpu_fused_fill.py -q -x -p no:cacheprovider 2>&1 | tail -2
: > gpurun_out/c1g.jsonl
for rep in 1 2 3 4; do timeout 300 python tools/probe.py c1 --tag c1 >> gpurun_out/c1g.jsonl 2>&1; done
python -c "
import json
for l in open('gpurun_out/c1g.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof']*1000,2), 'us/step', round(d['mcups_noprof']))
"
