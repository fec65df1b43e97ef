mkdir -p gpurun_out
for dbg in 0 4; do for sh in "0:0" "1:150"; do echo "== dbg $dbg SHAPE $sh" >> gpurun_out/trace_r.log; SCB_IC_DEBUG=$dbg SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 SHAPE=$sh timeout 300 python tools/ic_trace.py >> gpurun_out/trace_r.log 2>&1; done; done
for dbg in 0 4 6; do SCB_IC_DEBUG=$dbg CIN=96 COUT=96 SHAPES="1:96,1:150,2:42" timeout 300 python tools/layer_probe.py 2>&1 | sed "s/^/dbg=$dbg /" >> gpurun_out/probe_r.log; done
grep -v "^     " gpurun_out/trace_r.log; cat gpurun_out/probe_r.log
