mkdir -p gpurun_out
./tools/_mma_rate > gpurun_out/mma_rate.log 2>&1
for r in 1 0; do REORDER=$r CIN=96 COUT=96 LEVEL=0 timeout 300 python tools/layer_probe.py >> gpurun_out/probe_o.log 2>&1; done
CIN=96 COUT=96 LEVEL=0 REPS=2 NOWARM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_conv -s 3 -c 1 -o gpurun_out/r02o_fused96 python tools/layer_probe.py > gpurun_out/ncu_o.log 2>&1
cat gpurun_out/mma_rate.log gpurun_out/probe_o.log; tail -3 gpurun_out/ncu_o.log
