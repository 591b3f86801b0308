# multi-rank device guards: loopback tests, then C4 loopback timing A/B (BF_BATCH=0/1)
timeout 1200 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_nccl.py tests/test_gpu_iterate_loop.py -q -x -p no:cacheprovider 2>&1 | tail -3
for n in 2 8; do
  BF_BATCH=0 timeout 600 python tools/loopback_probe.py $n --steps 20 2>&1 | tail -1
  timeout 600 python tools/loopback_probe.py $n --steps 20 2>&1 | tail -1
done
