# round-2 evidence for the current build: ncu full capture of the stage kernel (both RK
# stages) on the bench workload -> profiles traffic; launch list of a short bench run;
# the bench line (native arm) and the reference arm; ghost-kernel capture
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vl_stage_kernel -c 2 -f -o gpurun_out/vl_final python tools/probe.py c4 --steps 1 --warmup 1 > gpurun_out/ncu_vl_final.log 2>&1
python profiles/ncu_summary.py gpurun_out/vl_final.ncu-rep --traffic 16777216 > gpurun_out/vl_final.json
cp profiles/stage_kernel_traffic.json gpurun_out/stage_kernel_traffic.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 3 --skip-cpu --skip-e2e --repeats 1 > /dev/null 2>&1
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 --flux roe --skip-cpu > gpurun_out/bench_final_roe.json 2>> gpurun_out/bench_final.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref_final.json 2> gpurun_out/ref_final.err; echo "ref rc=$?"
for c in c1 c2 c3; do timeout 300 python tools/probe.py $c --tag $c >> gpurun_out/info_final.jsonl 2>&1; done
timeout 300 python tools/probe.py c1 --flux roe --tag c1_roe >> gpurun_out/info_final.jsonl 2>&1
head -c 400 gpurun_out/bench_final.json
