ncu --set full --import-source on --clock-control none -k regex:attention_kernel_2sm -c 1 -o gpurun_out/r2_attn2sm_b python tools/attn_bench.py --reps 1 --runs 1 > gpurun_out/ncu_attn2sm.log 2>&1
