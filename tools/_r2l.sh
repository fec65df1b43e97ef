mkdir -p gpurun_out
for cfg in "96 96 0" "32 32 0" "64 64 0" "128 128 2"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="1:20,1:28,1:42,1:56,2:14,2:20,2:28,2:42,3:16" timeout 300 python tools/layer_probe.py >> gpurun_out/probe_l.log 2>&1; done
for sh in "1:28" "1:42" "2:14"; do SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=96 COUT=96 SHAPE=$sh timeout 300 python tools/ic_trace.py >> gpurun_out/trace_l.log 2>&1; done
cat gpurun_out/probe_l.log; grep -A4 "^CTA 0" gpurun_out/trace_l.log
