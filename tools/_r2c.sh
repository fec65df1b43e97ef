mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_reference_suite.py -q -x > gpurun_out/refsuite.log 2>&1; echo rc=$? >> gpurun_out/refsuite.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -n 3 gpurun_out/refsuite.log gpurun_out/gputest.log; head -12 gpurun_out/reference_suite.txt
