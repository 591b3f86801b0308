P="python tools/probe.py"
: > gpurun_out/g2.jsonl
for hide in 1 0; do
BF_HIDE_GHOSTS=$hide $P c4 --tag hide$hide >> gpurun_out/g2.jsonl 2>>gpurun_out/g2.err
done
$P box:128 --tag box128 >> gpurun_out/g2.jsonl 2>>gpurun_out/g2.err
BF_SPLIT_TILES=1 $P box:128 --tag box128_split >> gpurun_out/g2.jsonl 2>>gpurun_out/g2.err
BF_HIDE_GHOSTS=0 $P box:128 --tag box128_nohide >> gpurun_out/g2.jsonl 2>>gpurun_out/g2.err
timeout 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_overlap.py tests/test_gpu_loopback.py tests/test_gpu_parity.py tests/test_gpu_vl_split.py tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -15
