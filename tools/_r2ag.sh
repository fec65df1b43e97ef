mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/t_ag.log 2>&1; echo rc=$? >> gpurun_out/t_ag.log
tail -2 gpurun_out/t_ag.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_ag.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ag.log 2>&1
CIN=96 COUT=96 LEVEL=0 REPS=3 NOWARM=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:implicit -s 2 -c 1 -o gpurun_out/r02ag_fused96 python tools/layer_probe.py > gpurun_out/ncu_ag2.log 2>&1
CIN=64 COUT=64 LEVEL=1 REPS=3 NOWARM=1 SHAPES=5:48 timeout 600 ncu --set full --clock-control none --import-source on -k regex:implicit_conv_pair -s 1 -c 1 -o gpurun_out/r02ag_pair64 python tools/layer_probe.py > gpurun_out/ncu_ag3.log 2>&1
ls gpurun_out
