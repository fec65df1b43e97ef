mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
cat gpurun_out/e2e_probe.log
