timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_bwd_kernel -c 1 -o gpurun_out/ncu_abwd python tools/attn_bwd_bench.py --reps 1 --runs 1 > gpurun_out/ncu_abwd.log 2>&1
tail -3 gpurun_out/ncu_abwd.log
