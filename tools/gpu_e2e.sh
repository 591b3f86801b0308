# e2e variance: three bench runs (native arm, no CPU sample), blocks phase per run
for r in 1 2 3; do
  python bench.py --steps 20 --warmup 5 --skip-cpu > gpurun_out/e2e_$r.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/e2e_$r.json')); e=d['e2e']
print('$r', round(d['value']), 'e2e', round(e['value']), {k: round(v,4) for k,v in e['phases_s'].items() if k!='ctx_detail'}, [round(x,4) for x in e['phases_s']['ctx_detail']['blocks_s']])"
done
