nproc; free -g | head -2
python bench.py --steps 20 --warmup 5 > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/g3_ref.json 2> gpurun_out/g3_ref.err
python bench.py --steps 20 --warmup 5 --flux roe --skip-cpu --skip-e2e > gpurun_out/g3_roe.json 2>> gpurun_out/g3_bench.err
timeout 600 python -m pytest tests/test_bench_contract.py -q -m gpu 2>&1 | tail -3
