timeout 1500 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/t_c19.log 2>&1; echo tests; tail -2 gpurun_out/t_c19.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for d in 0 1; do SCB_DENSE_K1=$d timeout 300 python tools/pointwise_probe.py 2>&1 | tail -1; done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --layer-csv gpurun_out/r02cd_layers.csv > gpurun_out/bench_cd.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench_cd.log | cut -c1-200
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref_cd.log 2>&1; echo ref rc=$?; tail -1 gpurun_out/bench_ref_cd.log | cut -c1-200
timeout 600 python bench.py --model centerpoint --steps 20 --warmup 5 > gpurun_out/bench_cp_cd.log 2>&1; echo cp rc=$?; tail -1 gpurun_out/bench_cp_cd.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_cd.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cd.log 2>&1; echo ncu1 rc=$?
L1_REORDER=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:upconv -s 3 -c 1 -o gpurun_out/r02cd_upscatter python tools/up_probe.py > gpurun_out/ncu_cd2.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:upconv -s 3 -c 1 -o gpurun_out/r02cd_pointwise python tools/pointwise_probe.py > gpurun_out/ncu_cd3.log 2>&1; echo ncu3 rc=$?
