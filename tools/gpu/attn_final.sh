T="timeout 900"
$T python -m pytest tests/test_gpu_exec.py tests/test_gpu_baseline_sizes.py -m gpu -q -k "attention or llama or config2 or smoke or dispatch" 2>&1 | tail -2
$T python bench.py --no-offload-leg --no-cpu-baseline > gpurun_out/bench_attn.out 2>/dev/null
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attention_kernel_2sm -c 1 -o gpurun_out/r2b_attn python tools/attn_bench.py --reps 1 --runs 1 > /dev/null 2>&1
