TN_ATTN_EMU=3 PARITY_LOG=gpurun_out/par_emu3.jsonl python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "fused_attention" 2>&1 | tail -2
PARITY_LOG=gpurun_out/par_emu1.jsonl python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "fused_attention" 2>&1 | tail -2
for i in 1 2; do
TN_ATTN_1CTA=1 python tools/attn_bench.py; python tools/attn_bench.py; TN_ATTN_EMU=3 python tools/attn_bench.py; TN_ATTN_EMU=0 python tools/attn_bench.py
done
TN_ATTN_1CTA=1 python tools/attn_bench.py --causal 0; python tools/attn_bench.py --causal 0; TN_ATTN_EMU=3 python tools/attn_bench.py --causal 0
