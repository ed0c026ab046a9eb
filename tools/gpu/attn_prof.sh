cp abso/lib_prof.so paper_2405_16283_b200/lib/libturnip_b200.so
python tools/attn_bench.py --reps 1 --runs 1 > gpurun_out/prof_c.log 2>&1
python tools/attn_bench.py --reps 1 --runs 1 --causal 0 > gpurun_out/prof_nc.log 2>&1
