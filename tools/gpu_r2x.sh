# async node upload + deferred metric check: metric tests, e2e A/B (3 bench runs)
timeout 900 python -m pytest tests/test_gpu_device_metrics.py tests/test_gpu_memory.py tests/test_gpu_golden.py tests/test_gpu_parity.py -q -x -p no:cacheprovider 2>&1 | tail -2
for r in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --skip-cpu > gpurun_out/e2e_$r.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$r.json')); e=d['e2e']
print('$r', round(d['value']), 'e2e', round(e['value']), {k: round(v,4) for k,v in e['phases_s'].items() if k!='ctx_detail'}, e['phases_s']['ctx_detail'])"
done
