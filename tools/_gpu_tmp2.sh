mkdir -p gpurun_out/prof
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_r1c.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/prof/ncu_bench.log 2>&1
python tools/launch_summary.py gpurun_out/prof/launches_r1c.csv > gpurun_out/prof/launches_r1c.txt 2>&1
