timeout 900 python -m pytest "tests/test_gpu_parity_r2.py::test_c3_order_study_32_64_128_on_8_blocks" tests/test_gpu_iterate_loop.py -q -x -p no:cacheprovider 2>&1 | tail -3
: > gpurun_out/r2g_probe.jsonl
for c in c1 c2 c4; do python tools/probe.py $c --tag "$c" >> gpurun_out/r2g_probe.jsonl 2>&1; done
BF_BATCH=0 python tools/probe.py c1 --tag c1_nobatch >> gpurun_out/r2g_probe.jsonl 2>&1
BF_BATCH=0 python tools/probe.py c4 --tag c4_nobatch >> gpurun_out/r2g_probe.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2g_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'noprof', round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4))
"
