# final evidence of this build: GPU suite + smoke, ncu capture (traffic), launch list,
# bench (native: cold + repeated e2e), Roe line, reference arm, C1-C3 probes
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vl_stage_kernel -c 2 -f -o gpurun_out/vl_final3 python tools/probe.py c4 --steps 1 --warmup 1 > gpurun_out/ncu_vl_final3.log 2>&1
python profiles/ncu_summary.py gpurun_out/vl_final3.ncu-rep --traffic 16777216 > gpurun_out/vl_final3.json
cp profiles/stage_kernel_traffic.json gpurun_out/stage_kernel_traffic.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final3.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --repeats 1 > /dev/null 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final3.json 2> gpurun_out/bench_final3.err; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 --flux roe --skip-cpu --skip-e2e > gpurun_out/bench_final3_roe.json 2>> gpurun_out/bench_final3.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_final3.json 2> gpurun_out/ref_final3.err; echo "ref rc=$?"
for c in c1 c2 c3; do timeout 300 python tools/probe.py $c --tag $c >> gpurun_out/info_final3.jsonl 2>&1; done
python -c "
import json; d=json.load(open('gpurun_out/bench_final3.json')); e=d['e2e']
print(round(d['value']), d['roofline']['frac'], d['roofline']['traffic'], d['step_roofline_frac'], 'e2e', round(e['value']), 'cold', round(e['cold']['value']))"
