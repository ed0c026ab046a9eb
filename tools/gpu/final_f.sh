PARITY_LOG=gpurun_out/parity_r2f.jsonl timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu_f.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu_f.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_f.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke_f.log
timeout 900 python bench.py > gpurun_out/bench_f.out 2> gpurun_out/bench_f.err; echo bench_rc=$? >> gpurun_out/bench_f.err
