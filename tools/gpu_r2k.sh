# PDL + fused fill heuristic: full GPU suite, then C1/C2/C4 timing A/B
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -4
: > gpurun_out/r2k_probe.jsonl
for c in c1 c2 c4; do
  BF_PDL=0 BF_FUSED_FILL=0 timeout 300 python tools/probe.py $c --tag "${c}_base" >> gpurun_out/r2k_probe.jsonl 2>&1
  BF_FUSED_FILL=0 timeout 300 python tools/probe.py $c --tag "${c}_pdl" >> gpurun_out/r2k_probe.jsonl 2>&1
  timeout 300 python tools/probe.py $c --tag "${c}_default" >> gpurun_out/r2k_probe.jsonl 2>&1
done
BF_FUSED_FILL=1 timeout 300 python tools/probe.py c1 --tag "c1_pdl_fill1" >> gpurun_out/r2k_probe.jsonl 2>&1
python -c "
import json
for l in open('gpurun_out/r2k_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'noprof', round(d['ms_per_step_noprof'],4), 'mcups_noprof', round(d['mcups_noprof']), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4))
"
