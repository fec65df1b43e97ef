mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_voxelize.py tests/test_autotune.py -q -m gpu > gpurun_out/t_f.log 2>&1; echo rc=$? >> gpurun_out/t_f.log
for l1 in 0 1; do
  for cfg in "96 96" "32 32" "64 64" "128 128" "256 256"; do set -- $cfg; SCB_IC_L1=$l1 CIN=$1 COUT=$2 SHAPES="1:64,1:96,1:128,2:28,2:42,2:56,3:16,3:24" timeout 300 python tools/layer_probe.py >> gpurun_out/probe_f.log 2>&1; done
done
for cfg in "128 128 2" "256 256 3" "256 256 4"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="1:64,1:96,2:42,2:56" timeout 300 python tools/layer_probe.py >> gpurun_out/probe_f.log 2>&1; done
tail -n 3 gpurun_out/t_f.log; cat gpurun_out/probe_f.log
