for i in 1 2 3 4; do
  PYTHONFAULTHANDLER=1 timeout -s SIGABRT 240 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_am$i.log 2>&1
  echo "run $i rc=$?"; tail -c 300 gpurun_out/bench_am$i.log | head -c 300; echo
done
