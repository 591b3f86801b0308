timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider --durations=8 > gpurun_out/r2f_tests.log 2>&1; echo "tests rc=$?"
tail -16 gpurun_out/r2f_tests.log
: > gpurun_out/r2f_probe.jsonl
for c in c1 c2 c3 c4; do python tools/probe.py $c --tag "$c" >> gpurun_out/r2f_probe.jsonl 2>&1; done
BF_BATCH=0 python tools/probe.py c1 --tag c1_nobatch >> gpurun_out/r2f_probe.jsonl 2>&1
python tools/probe.py c1 --flux roe --tag c1_roe >> gpurun_out/r2f_probe.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2f_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4), 'mcups', round(d['mcups']))
"
