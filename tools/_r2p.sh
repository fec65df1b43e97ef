mkdir -p gpurun_out
CIN=96 COUT=96 LEVEL=0 REPS=3 NOWARM=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit -s 2 -c 1 -o gpurun_out/r02p_fused96 python tools/layer_probe.py > gpurun_out/ncu_p.log 2>&1
tail -3 gpurun_out/ncu_p.log; ls -la gpurun_out
