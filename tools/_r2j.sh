mkdir -p gpurun_out
timeout 600 python tools/e2e_probe.py > gpurun_out/e2e_probe.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
cat gpurun_out/e2e_probe.log; tail -3 gpurun_out/gputest.log
