T="timeout 60"
$T python -m pytest tests/test_gpu_exec.py -m gpu -x -q -k "fused_attention" 2>&1 | tail -1
for i in 1 2 3; do
TN_ATTN_PAIR=0 $T python tools/attn_bench.py; $T python tools/attn_bench.py
done
$T python tools/attn_bench.py --causal 0
