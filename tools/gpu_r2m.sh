# A/B: DevBlock in shared memory (smemb) vs base; ghost items per thread (wave fit vs 4)
bash tools/ab_probe.sh c4 base smemb
: > gpurun_out/ipt.jsonl
for rep in 1 2; do
for ipt in 4 3 0; do
  if [ $ipt = 0 ]; then unset BF_GHOST_IPT; else export BF_GHOST_IPT=$ipt; fi
  timeout 300 python tools/probe.py c4 --tag "ipt$ipt" >> gpurun_out/ipt.jsonl 2>&1
done; done
unset BF_GHOST_IPT
python -c "
import json
for l in open('gpurun_out/ipt.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof'],4), 'ghost', round(d['ghost_ms'],4), 'stage', round(d['stage_ms'],4))
"
