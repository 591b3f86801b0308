# kc sweep (box 128^3 forced split = the 8-GPU strong-scaling block; C4) and precision variants
: > gpurun_out/kc.jsonl
for kc in 8 10 11 13 15 16 22 32; do
BF_KC=$kc BF_SPLIT_TILES=1 python tools/probe.py box:128 --tag "box128s_kc$kc" >> gpurun_out/kc.jsonl 2>>gpurun_out/kc.err
BF_KC=$kc python tools/probe.py box:128 --tag "box128_kc$kc" >> gpurun_out/kc.jsonl 2>>gpurun_out/kc.err
done
for kc in 16 22 26 29 32 43; do
BF_KC=$kc python tools/probe.py c4 --tag "c4_kc$kc" >> gpurun_out/kc.jsonl 2>>gpurun_out/kc.err
done
for v in rcpfull rcpn2; do
BFGPU_LIB=paper_2012_02925_b200/libbfgpu_$v.so python tools/probe.py c4 --tag "c4_$v" >> gpurun_out/kc.jsonl 2>>gpurun_out/kc.err
done
python tools/probe.py c4 --tag "c4_base" >> gpurun_out/kc.jsonl 2>>gpurun_out/kc.err
python -c "
import json
for l in open('gpurun_out/kc.jsonl'):
    d=json.loads(l); print(d['tag'], round(d['stage_ms'],4), round(d['stage_hbm_frac'],3), round(d['ms_per_step'],4))
"
