PARITY_LOG=gpurun_out/parity_r2g.jsonl timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_g.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_g.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_g2.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_g2.log
timeout 900 python bench.py > gpurun_out/bench_g.out 2> gpurun_out/bench_g.err; echo bench_rc=$? >> gpurun_out/bench_g.err
