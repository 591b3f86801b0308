set -x
timeout 800 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -1 gpurun_out/gputests.log
for g in 0 1; do
  BF_GRAPH=$g timeout 300 python bench.py --skip-cpu --skip-e2e --steps 20 > gpurun_out/g_c4_$g.log 2>&1
  BF_GRAPH=$g timeout 300 python bench.py --skip-cpu --workload c1 --steps 200 > gpurun_out/g_c1_$g.log 2>&1
  BF_GRAPH=$g timeout 300 python bench.py --skip-cpu --workload c2 --steps 50 > gpurun_out/g_c2_$g.log 2>&1
done
