# A/B: L2 evict_last hint on the band cells (l2a: others normal, l2b: others evict_first),
# with and without a persisting-L2 set-aside
bash tools/ab_probe.sh c4 base l2a l2b
: > gpurun_out/l2p.jsonl
for mb in 32 64; do for v in l2a l2b; do
  BF_L2_PERSIST_MB=$mb BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_$v.so timeout 300 python tools/probe.py c4 --tag "${v}_persist$mb" >> gpurun_out/l2p.jsonl 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/l2p.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4))
"
