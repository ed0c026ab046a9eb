for e in 1 2 0 1 2; do TN_ATTN_EMU=$e timeout 120 python tools/attn_bench.py --reps 8 --runs 3 2>&1 | tail -1; done
TN_ATTN_EMU=2 timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "fused_attention_parity" 2>&1 | tail -1
