mkdir -p gpurun_out
for cfg in "96 96" "32 32" "64 64" "128 128"; do set -- $cfg; for dbg in 0 1 2 3 0; do SCB_IC_DEBUG=$dbg CIN=$1 COUT=$2 timeout 300 python tools/layer_probe.py 2>&1 | sed "s/^/dbg=$dbg /" >> gpurun_out/probe_m.log; done; done
cat gpurun_out/probe_m.log
