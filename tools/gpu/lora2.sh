# config 4: recomputed norms / backward recompute prefetch, plan-order default
timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_baseline_sizes.py -m gpu -q -k "lora or config4 or dispatch or order" 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --dump gpurun_out/lora_dump2.json 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --bwd-prefetch 1 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --no-recompute-norms 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --exec-cfg '{"tie_break": "fifo"}' 2>&1 | tail -1
