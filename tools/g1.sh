set -x
P="python tools/probe.py"
$P c4 --tag base > gpurun_out/g1.jsonl 2>gpurun_out/g1.err
$P c4 --flux roe --tag roe >> gpurun_out/g1.jsonl 2>>gpurun_out/g1.err
$P box:128 --tag box128 >> gpurun_out/g1.jsonl 2>>gpurun_out/g1.err
BF_SPLIT_TILES=1 $P box:128 --tag box128_split >> gpurun_out/g1.jsonl 2>>gpurun_out/g1.err
BF_KC=16 $P box:128 --tag box128_kc16 >> gpurun_out/g1.jsonl 2>>gpurun_out/g1.err
$P c1 --tag c1 >> gpurun_out/g1.jsonl 2>>gpurun_out/g1.err
