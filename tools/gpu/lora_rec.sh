timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -q -k "gemm or lora or graph_mode or blockwise" 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 2>&1 | tail -1
