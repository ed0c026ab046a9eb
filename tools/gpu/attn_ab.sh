T="timeout 60"
PARITY_LOG=gpurun_out/par_pers.jsonl TN_ATTN_PAIR=1 $T python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "fused_attention" 2>&1 | tail -2
$T python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "fused_attention" 2>&1 | tail -1
for i in 1 2; do
$T python tools/attn_bench.py; TN_ATTN_PAIR=1 $T python tools/attn_bench.py; TN_ATTN_PAIR=1 TN_ATTN_EMU=0 $T python tools/attn_bench.py
done
TN_ATTN_1CTA=1 $T python tools/attn_bench.py --causal 0; $T python tools/attn_bench.py --causal 0
