timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "attention_bwd" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -20
for s in 0 1 0 1; do TN_ATTN_BWD_SPIN=$s timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -1; done
