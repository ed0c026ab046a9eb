# config 4 with the fused attention backward as the default LoRA graph
PARITY_LOG=gpurun_out/parity_fused.jsonl timeout 1200 python -m pytest tests/test_gpu_exec.py tests/test_gpu_baseline_sizes.py -m gpu -q -k "lora or config4 or attention_bwd or graph_mode or elision or fused_attention" 2>&1 | grep -E "passed|failed|Error|assert" | head -20
timeout 600 python tools/bench_lora.py --steps 3 --compare --dump gpurun_out/lora_dump_fused.json 2>&1 | tail -1
