timeout 900 python -m pytest tests/test_gpu_upscatter.py -x -q --timeout 240 > gpurun_out/t_c23.log 2>&1; echo tests; tail -2 gpurun_out/t_c23.log
for d in 0 2 6; do SCB_UP_DEBUG=$d EPI=1 L1_REORDER=1 timeout 300 python tools/up_probe.py 2>&1 | tail -1; echo "debug=$d"; done
SCB_UP_DEBUG=2 L1_REORDER=1 timeout 600 ncu --metrics gpu__time_duration.sum -k regex:upconv -s 3 -c 1 python tools/up_probe.py 2>&1 | grep -i "duration"
L1_REORDER=1 timeout 600 ncu --metrics gpu__time_duration.sum -k regex:upconv -s 3 -c 1 python tools/up_probe.py 2>&1 | grep -i "duration"
