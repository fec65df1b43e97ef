mkdir -p gpurun_out
for sh in "4:0" "5:48"; do echo "== SHAPE $sh" >> gpurun_out/trace_v.log; TRACE_CTAS=0,2 SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 SHAPE=$sh timeout 120 python tools/ic_trace.py >> gpurun_out/trace_v.log 2>&1; done
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/t_v.log 2>&1; echo rc=$? >> gpurun_out/t_v.log
grep -v "^     " gpurun_out/trace_v.log; tail -3 gpurun_out/t_v.log
