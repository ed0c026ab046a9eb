# fused attention backward: parity, micro-benchmark, LoRA step with it
timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "attention_bwd or fused_attention_parity" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -20
timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -2
timeout 120 python tools/attn_bwd_bench.py --causal 0 --reps 3 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --fused-attention 1 2>&1 | tail -1
