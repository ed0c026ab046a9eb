python tools/attn_bench.py > gpurun_out/attn_base.json 2>&1
python tools/attn_bench.py --causal 0 >> gpurun_out/attn_base.json 2>&1
TN_ATTN_DBG=gpurun_out/attn_dbg_causal.txt python tools/attn_bench.py --reps 1 --runs 3 > gpurun_out/attn_dbg.log 2>&1
TN_ATTN_DBG=gpurun_out/attn_dbg_noncausal.txt python tools/attn_bench.py --reps 1 --runs 3 --causal 0 >> gpurun_out/attn_dbg.log 2>&1
