timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/t_an.log 2>&1; echo tests rc=$?
ps aux | grep -c python
PYTHONFAULTHANDLER=1 timeout -s SIGABRT 300 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_an.log 2>&1
echo "bench rc=$?"; grep -v "^  File \"/opt" gpurun_out/bench_an.log | tail -25 | cut -c1-300
