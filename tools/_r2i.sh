mkdir -p gpurun_out
timeout 600 python tools/d2h_probe.py > gpurun_out/d2h_probe.log 2>&1
for cfg in "96 96 0:0" "32 32 0:0" "96 96 1:42" "256 256 0:0"; do set -- $cfg; SCB_LIB_NAME=libsparseconv_b200_trace.so CIN=$1 COUT=$2 SHAPE=$3 timeout 300 python tools/ic_trace.py >> gpurun_out/ic_trace.log 2>&1; done
cat gpurun_out/d2h_probe.log gpurun_out/ic_trace.log
