mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_minkunet.py tests/test_gpu_reorder.py -q -x > gpurun_out/t_k.log 2>&1; echo rc=$? >> gpurun_out/t_k.log
for cfg in "96 96 0" "128 96 0" "32 32 0" "64 64 0" "128 128 2" "256 256 3" "256 256 4"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 timeout 300 python tools/layer_probe.py >> gpurun_out/probe_k.log 2>&1; done
for cfg in "96 96" "32 32"; do set -- $cfg; SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=$1 COUT=$2 timeout 300 python tools/ic_trace.py >> gpurun_out/trace_k.log 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_k.log 2>&1
tail -n 3 gpurun_out/t_k.log; cat gpurun_out/probe_k.log; head -12 gpurun_out/trace_k.log; tail -1 gpurun_out/bench_k.log | cut -c1-300
