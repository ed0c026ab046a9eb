# EMU sweep of the pair attention kernel; values 2 / 3 need the attention_kernel_2sm<2> / <3>
# instantiations and dispatch (built for the r2f sweep, not kept: 1 is the fastest)
for r in 1 2; do for e in 1 2 3 0; do TN_ATTN_EMU=$e python tools/attn_bench.py | sed "s/^/emu$e /"; done; done > gpurun_out/attn_emu.txt 2>&1
for e in 1 2; do TN_ATTN_EMU=$e python tools/attn_bench.py --causal 0 | sed "s/^/nc emu$e /"; done >> gpurun_out/attn_emu.txt 2>&1
