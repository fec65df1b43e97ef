mkdir -p gpurun_out
for sh in "0:0" "1:96" "1:150" "2:30"; do echo "== SHAPE $sh" >> gpurun_out/trace_q.log; SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 SHAPE=$sh timeout 300 python tools/ic_trace.py >> gpurun_out/trace_q.log 2>&1; done
for dbg in 0 1 2 3; do SCB_IC_DEBUG=$dbg CIN=96 COUT=96 SHAPES="1:96,1:150,2:30,2:42,3:24" timeout 300 python tools/layer_probe.py 2>&1 | sed "s/^/dbg=$dbg /" >> gpurun_out/probe_q.log; done
cat gpurun_out/trace_q.log gpurun_out/probe_q.log
