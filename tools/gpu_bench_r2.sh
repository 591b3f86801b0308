# round-2 bench refresh: bench line, reference arm, ncu launch lists (small outputs)
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 --flux roe --skip-cpu > gpurun_out/bench_r2_roe.json 2>> gpurun_out/bench_r2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_r2.json 2> gpurun_out/ref_r2.err; echo "ref rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --repeats 1 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_r2_c1.csv python tools/probe.py c1 --steps 3 --warmup 3 > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vl_stage_kernel -c 2 -f -o gpurun_out/vl_r2 python tools/probe.py c4 --steps 1 --warmup 0 > gpurun_out/ncu_vl.log 2>&1; echo "ncu vl rc=$?"
ls -la gpurun_out/
