TN_ATTN_OCC=1 python tools/attn_bench.py --reps 1 --runs 1 2>&1 | grep -v Warn | head -3
ncu --set full --import-source on --clock-control none -k regex:attention_kernel_2sm -c 1 -o gpurun_out/r2_attn2sm python tools/attn_bench.py --reps 1 --runs 1 > gpurun_out/ncu_attn2sm.log 2>&1
tail -3 gpurun_out/ncu_attn2sm.log
