#!/bin/bash
# A/B timing of library variants on the 2D workloads (C1, C2): tools/abl2d.sh name...
for v in "$@"; do
  lib=paper_2012_02925_b200/libbfgpu.so
  [ "$v" != "base" ] && lib=paper_2012_02925_b200/libbfgpu_$v.so
  for w in c1 c2; do
    BFGPU_LIB=$PWD/$lib timeout 300 python bench.py --skip-cpu --skip-e2e --workload $w --steps 50 > gpurun_out/abl2d_${v}_$w.log 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abl2d_${v}_$w.log').read().strip().splitlines()[-1]); print('$v $w', round(d['value'],1), round(d['ms_per_step'],4), round(d['roofline']['avg_launch_ms'],5), round(d['roofline']['frac'],4))" >> gpurun_out/abl2d.txt
  done
done
