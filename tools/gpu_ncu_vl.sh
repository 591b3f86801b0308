# ncu --set full of the C4 stage kernel (both stage variants) and the ghost kernel
timeout 900 ncu --set full --import-source on --clock-control none -k regex:vl_stage_kernel -c 2 -f -o gpurun_out/vl_r2b python tools/probe.py c4 --steps 1 --warmup 1 > gpurun_out/ncu_vl.log 2>&1; echo "ncu vl rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ghost_kernel -c 1 -f -o gpurun_out/ghost_r2b python tools/probe.py c4 --steps 1 --warmup 1 > gpurun_out/ncu_ghost.log 2>&1; echo "ncu ghost rc=$?"
ls -la gpurun_out/*.ncu-rep
