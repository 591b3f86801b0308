# bench e2e (cold + repeated call) on a fresh box: first run and a second run
timeout 900 python -m pytest tests/test_gpu_device_metrics.py tests/test_bench_contract.py -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2; do
  python bench.py --steps 20 --warmup 5 > gpurun_out/e2e_$r.json 2>gpurun_out/e2e_$r.err
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$r.json')); e=d['e2e']
print('$r', round(d['value']), 'e2e', round(e['value']), 'cold', round(e['cold']['value']), {k: round(v,4) for k,v in e['phases_s'].items() if k!='ctx_detail'}, {k: round(v,4) for k,v in e['cold']['phases_s'].items() if k!='ctx_detail'})"
done
