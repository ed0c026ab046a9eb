timeout 900 python bench.py > gpurun_out/bench.out 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-leg > /dev/null 2>&1
