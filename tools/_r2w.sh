mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/t_w.log 2>&1; echo rc=$? >> gpurun_out/t_w.log
tail -3 gpurun_out/t_w.log
for cfg in "96 96 0" "32 32 0" "64 64 1" "128 128 2"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="2:0,4:0,5:0,4:48,5:24,5:48" timeout 120 python tools/layer_probe.py >> gpurun_out/probe_w.log 2>&1; done
cat gpurun_out/probe_w.log
for sh in "4:0" "5:48"; do echo "== SHAPE $sh" >> gpurun_out/trace_w.log; TRACE_CTAS=0,2 SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 SHAPE=$sh timeout 120 python tools/ic_trace.py >> gpurun_out/trace_w.log 2>&1; done
grep -v "^     " gpurun_out/trace_w.log | grep -v "CTA 2" 
