# A/B: lamz in smem; k-chunk sweep on the smem-block build
bash tools/ab_probe.sh c4 base lamz
: > gpurun_out/kc2.jsonl
for kc in 24 32 40 48; do
  BF_KC=$kc timeout 300 python tools/probe.py c4 --tag "kc$kc" >> gpurun_out/kc2.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/kc2.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4))
"
