mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gputest.log 2>&1; echo rc=$? >> gpurun_out/gputest.log
for cfg in "A SCB_REORDER=1" "B SCB_REORDER=0"; do
  set -- $cfg
  env $2 timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_$1.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
tail -n 3 gpurun_out/gputest.log; tail -n 2 gpurun_out/bench_*.log
