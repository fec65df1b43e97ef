mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_reference_models.py tests/test_gpu_parity.py -q -k "reference or chain or duplicate" > gpurun_out/reftests.log 2>&1; echo rc=$? >> gpurun_out/reftests.log
for cfg in "96 96" "128 96" "32 32" "64 64"; do set -- $cfg; CIN=$1 COUT=$2 timeout 300 python tools/layer_probe.py >> gpurun_out/probe.log 2>&1; done
CIN=96 COUT=96 REORDER=0 timeout 300 python tools/layer_probe.py >> gpurun_out/probe.log 2>&1
CIN=96 COUT=96 NOWARM=1 REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_conv -s 1 -c 1 -o gpurun_out/ic96 python tools/layer_probe.py > gpurun_out/ncu_ic96.log 2>&1
tail -n 4 gpurun_out/reftests.log; cat gpurun_out/probe.log
