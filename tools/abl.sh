#!/bin/bash
# A/B timing of library variants on the bench workload: tools/abl.sh name...
# (one untimed run first: the first bench on a fresh box reads a few % slow)
timeout 300 python bench.py --skip-cpu --skip-e2e --steps 5 > /dev/null 2>&1
for v in "$@"; do
  lib=paper_2012_02925_b200/libbfgpu.so
  [ "$v" != "base" ] && lib=paper_2012_02925_b200/libbfgpu_$v.so
  BFGPU_LIB=$PWD/$lib timeout 300 python bench.py --skip-cpu --skip-e2e --steps 20 > gpurun_out/abl_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abl_$v.log').read().strip().splitlines()[-1]); print('$v', round(d['value']), round(d['roofline']['avg_launch_ms'],4), round(d['roofline']['frac'],4), 'ghost', round(d['kernel_ms']['ghost_fill'],3))" >> gpurun_out/abl.txt
done
