mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_reference_suite.py -q -x > gpurun_out/refsuite.log 2>&1; echo rc=$? >> gpurun_out/refsuite.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --layer-csv gpurun_out/layers.csv > gpurun_out/bench_L.log 2>&1
tail -n 5 gpurun_out/refsuite.log; head -3 gpurun_out/reference_suite.txt
