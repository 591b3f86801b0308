# copy-only ghost push: bitwise check vs the ghost kernel, then C4 A/B
python tools/push_check.py gpurun_out/pc_base.npz 6
BF_PUSH=1 BF_PUSH_COPY=1 BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_push.so python tools/push_check.py gpurun_out/pc_push.npz 6
python -c "
import numpy as np
a=np.load('gpurun_out/pc_base.npz'); b=np.load('gpurun_out/pc_push.npz')
bad=[k for k in a.files if not np.array_equal(a[k], b[k])]
print('push bitwise:', 'OK' if not bad else bad[:10])
"
: > gpurun_out/push.jsonl
for rep in 1 2; do
  timeout 300 python tools/probe.py c4 --tag base >> gpurun_out/push.jsonl 2>&1
  BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_push.so timeout 300 python tools/probe.py c4 --tag pushlib_off >> gpurun_out/push.jsonl 2>&1
  BF_PUSH=1 BF_PUSH_COPY=1 BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_push.so timeout 300 python tools/probe.py c4 --tag push_copy >> gpurun_out/push.jsonl 2>&1
  BF_PUSH=1 BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu_push.so timeout 300 python tools/probe.py c4 --tag push_all >> gpurun_out/push.jsonl 2>&1
done
python -c "
import json
for l in open('gpurun_out/push.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d['tag'], round(d['ms_per_step_noprof'],4), 'stage', round(d['stage_ms'],4), 'ghost', round(d['ghost_ms'],4))
"
