# compute-sanitizer on small cases of every kernel family (memcheck, synccheck, racecheck)
export BF_FUSED_FILL=1
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/probe.py c4:6 --steps 2 --warmup 1 > gpurun_out/san_${tool}_c4.log 2>&1; echo "$tool c4:6 rc=$?"
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 python tools/probe.py c1 --steps 2 --warmup 1 > gpurun_out/san_${tool}_c1.log 2>&1; echo "$tool c1 rc=$?"
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python tools/probe.py c4:6 --flux roe --steps 2 --warmup 1 > gpurun_out/san_memcheck_roe.log 2>&1; echo "memcheck roe rc=$?"
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python tools/probe.py c4:6 --precision exact --steps 2 --warmup 1 > gpurun_out/san_memcheck_exact.log 2>&1; echo "memcheck exact rc=$?"
tail -3 gpurun_out/san_*.log
