mkdir -p gpurun_out
python -m pytest tests/test_gpu_reorder.py tests/test_gpu_parity.py -x -q > gpurun_out/t_reorder.log 2>&1; echo rc=$? >> gpurun_out/t_reorder.log
for cfg in "A SCB_REORDER=1" "B SCB_REORDER=0" "C SCB_IC_INTERLEAVE=0"; do
  set -- $cfg
  env $2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_$1.log 2>&1
done
python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
tail -3 gpurun_out/t_reorder.log gpurun_out/gputest.log
