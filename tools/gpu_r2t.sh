# forced interior/boundary split (the multi-GPU launch structure) on C4 and box:128/256
: > gpurun_out/split.jsonl
for c in c4 box:256 box:128; do
  timeout 300 python tools/probe.py $c --tag "${c}_one" >> gpurun_out/split.jsonl 2>&1
  BF_SPLIT_TILES=1 timeout 300 python tools/probe.py $c --tag "${c}_split" >> gpurun_out/split.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/split.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'frac', round(d['stage_hbm_frac'],4))
"
