T="timeout 60"
for i in 1 2 3; do
$T python tools/attn_bench.py; TN_ATTN_EMU=2 $T python tools/attn_bench.py; TN_ATTN_EMU=0 $T python tools/attn_bench.py
done
