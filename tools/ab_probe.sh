#!/bin/bash
# A/B of library variants with tools/probe.py (alternating, 3 rounds):
#   tools/ab_probe.sh CASE name...   (name "base" = libbfgpu.so, else libbfgpu_<name>.so)
case=$1; shift
out=gpurun_out/ab_${case//:/_}.jsonl
: > $out
BFGPU_LIB=$PWD/paper_2012_02925_b200/libbfgpu.so timeout 300 python tools/probe.py $case --steps 5 > /dev/null 2>&1
for rep in 1 2 3; do
  for v in "$@"; do
    lib=paper_2012_02925_b200/libbfgpu.so
    [ "$v" != "base" ] && lib=paper_2012_02925_b200/libbfgpu_$v.so
    BFGPU_LIB=$PWD/$lib timeout 300 python tools/probe.py $case --tag "$v" >> $out 2>&1
  done
done
python - "$out" <<'PY'
import json, sys, collections
d = collections.defaultdict(list)
for l in open(sys.argv[1]):
    try: r = json.loads(l)
    except Exception: print(l[:200]); continue
    d[r['tag']].append((r['ms_per_step_noprof'], r['stage_ms'], r['ghost_ms']))
for t, v in d.items():
    print(t, 'noprof', [round(x[0], 4) for x in v], 'stage', [round(x[1], 4) for x in v], 'ghost', [round(x[2], 4) for x in v])
PY
