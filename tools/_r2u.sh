mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_pair.py -q -x > gpurun_out/t_u.log 2>&1; echo rc=$? >> gpurun_out/t_u.log
tail -30 gpurun_out/t_u.log
for cfg in "96 96 0" "32 32 0" "64 64 1" "128 128 2" "256 256 3"; do set -- $cfg; CIN=$1 COUT=$2 LEVEL=$3 SHAPES="2:0,1:0,4:0,5:0,4:48,4:96,5:24,5:48" timeout 120 python tools/layer_probe.py >> gpurun_out/probe_u.log 2>&1; done
cat gpurun_out/probe_u.log
