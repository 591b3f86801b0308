# smem DevBlock default: GPU suite, C4 VL + Roe A/B vs the register copy, bench line
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/ab_probe.sh c4 base nosmemb
: > gpurun_out/roe_ab.jsonl
for rep in 1 2; do for v in base nosmemb; do
  lib=paper_2012_02925_b200/libbfgpu.so; [ $v != base ] && lib=paper_2012_02925_b200/libbfgpu_$v.so
  BFGPU_LIB=$PWD/$lib timeout 300 python tools/probe.py c4 --flux roe --tag "roe_$v" >> gpurun_out/roe_ab.jsonl 2>&1
done; done
python -c "
import json
for l in open('gpurun_out/roe_ab.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4))
"
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2n.json 2> gpurun_out/bench_r2n.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/bench_r2n.json'))
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['step_roofline_frac'], d['e2e']['value'])"
