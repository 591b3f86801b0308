#!/bin/bash
# stage-kernel time vs k-chunk (BF_KC): tools/kc_sweep.sh 8 16 24 32
for kc in "$@"; do
  BF_KC=$kc timeout 300 python bench.py --skip-cpu --skip-e2e --steps 20 > gpurun_out/kc_$kc.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/kc_$kc.log').read().strip().splitlines()[-1]); print('kc', $kc, round(d['value']), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4))" >> gpurun_out/kc.txt
done
