PARITY_LOG=gpurun_out/parity_rope.jsonl timeout 900 python -m pytest tests/test_gpu_exec.py tests/test_gpu_baseline_sizes.py -m gpu -q -k "lora or config4 or attention_bwd or graph_mode" 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 600 python tools/bench_lora.py --steps 3 --dump gpurun_out/lora_dump_rope.json 2>&1 | tail -1 | cut -c1-1500
timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -1
