# A/B: 2 CTAs/SM (32x8 tiles) on the smem-block build
bash tools/ab_probe.sh c4 base tj8
: > gpurun_out/tj8kc.jsonl
for kc in 16 24 48; do
  BF_KC=$kc BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_tj8.so timeout 300 python tools/probe.py c4 --tag "tj8_kc$kc" >> gpurun_out/tj8kc.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/tj8kc.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4))
"
