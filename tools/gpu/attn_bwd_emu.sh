timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "attention_bwd or fused_attention_parity" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -20
for e in 0 1 2; do TN_ATTN_BWD_EMU=$e timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -1; done
TN_ATTN_BWD_EMU=2 timeout 120 python tools/attn_bwd_bench.py --causal 0 --reps 3 2>&1 | tail -1
