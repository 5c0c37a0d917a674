set -u
bash tools/bench_all.sh > gpurun_out/bench_all.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r02_launches_config5_k4a.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
sh tools/ncu_capture.sh config5 > gpurun_out/ncu_capture.log 2>&1
sh tools/ncu_capture.sh config2 >> gpurun_out/ncu_capture.log 2>&1
cat gpurun_out/bench_all.log
