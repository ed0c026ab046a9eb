timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "attention_bwd" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -20
timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -1
timeout 120 python tools/attn_bwd_bench.py --causal 0 --reps 3 2>&1 | tail -1
