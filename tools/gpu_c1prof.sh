timeout 600 ncu --set full --clock-control none -k regex:"ghost_kernel|vl_stage_kernel|guard_kernel" -s 20 -c 5 -f -o gpurun_out/c1_r2 python tools/probe.py c1 --steps 5 --warmup 5 > gpurun_out/c1prof.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out
