PARITY_LOG=gpurun_out/parity_r2f.jsonl timeout 1800 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.out 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.out 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d_launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-offload-leg > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_bwd_kernel -c 1 -o gpurun_out/ncu_abwd_final python tools/attn_bwd_bench.py --reps 1 --runs 1 > /dev/null 2>&1
timeout 300 python tools/attn_bwd_bench.py > gpurun_out/attn_bwd_bench.json 2>&1
