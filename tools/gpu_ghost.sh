: > gpurun_out/ghost.jsonl
for v in "" gm6 gm8; do
  lib=paper_2012_02925_b200/libbfgpu${v:+_$v}.so
  for c in c4 c1; do BFGPU_LIB=$lib python tools/probe.py $c --tag "${c}_${v:-base}" >> gpurun_out/ghost.jsonl 2>&1; done
done
python -c "
import json
for l in open('gpurun_out/ghost.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:200]); continue
    print(d['tag'], 'noprof', round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4))
"
timeout 600 ncu --set full --clock-control none -k regex:ghost_kernel -c 1 -f -o gpurun_out/ghost_r2 python tools/probe.py c4 --steps 1 --warmup 0 > /dev/null 2>&1; echo "ncu rc=$?"
