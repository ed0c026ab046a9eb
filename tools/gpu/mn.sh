# MN-major operands: GEMM / LoRA parity, then config-4 step with and without transposes
timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_baseline_sizes.py -m gpu -q -k "gemm or lora or graph_mode or config4" 2>&1 | grep -E "FAILED|passed|failed|^E " | head -30
timeout 600 python tools/bench_lora.py --steps 3 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --no-mn-major 2>&1 | tail -1
