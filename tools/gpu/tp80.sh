timeout 1200 python tools/bench_tp.py --layers 80 --cap-gib 16 --steps 2 --execution events > gpurun_out/tp80_events.out 2>&1
timeout 1200 python tools/bench_tp.py --layers 80 --cap-gib 16 --steps 2 --execution graph > gpurun_out/tp80_graph.out 2>&1
