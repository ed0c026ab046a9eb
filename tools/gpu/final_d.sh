PARITY_LOG=gpurun_out/parity_r2e.jsonl timeout 1800 python -m pytest tests -m gpu -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.out 2> gpurun_out/bench.err; echo bench_rc=$? >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.out 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2e_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-leg --no-other-configs > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_kernel_2sm -c 1 -o gpurun_out/r2e_attn python tools/attn_bench.py --reps 1 --runs 1 > /dev/null 2>&1
