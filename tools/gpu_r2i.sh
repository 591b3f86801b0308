# fused ghost fill: parity tests, then A/B timing on C1..C4 and a fill-CTA sweep on C4
timeout 900 python -m pytest tests/test_gpu_fused_fill.py tests/test_gpu_graph.py tests/test_gpu_iterate_loop.py -q -x -p no:cacheprovider 2>&1 | tail -5
: > gpurun_out/r2i_probe.jsonl
for c in c1 c2 c4; do
  BF_FUSED_FILL=0 timeout 300 python tools/probe.py $c --tag "${c}_sep" >> gpurun_out/r2i_probe.jsonl 2>&1
  timeout 300 python tools/probe.py $c --tag "${c}_fused" >> gpurun_out/r2i_probe.jsonl 2>&1
done
for n in 8 24 32; do
  BF_FILL_CTAS=$n timeout 300 python tools/probe.py c4 --tag "c4_fused_n$n" >> gpurun_out/r2i_probe.jsonl 2>&1
done
for n in 4 8 32; do
  BF_FILL_CTAS=$n timeout 300 python tools/probe.py c2 --tag "c2_fused_n$n" >> gpurun_out/r2i_probe.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/r2i_probe.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], 'ms/step', round(d['ms_per_step'],4), 'noprof', round(d['ms_per_step_noprof'],4), 'mcups_noprof', round(d['mcups_noprof']), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4), 'red', round(d['reduce_ms'],4))
"
