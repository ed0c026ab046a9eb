python tools/attn_bench.py > gpurun_out/attn_ab2.json 2>&1
python tools/attn_bench.py --causal 0 >> gpurun_out/attn_ab2.json 2>&1
python tools/attn_bench.py >> gpurun_out/attn_ab2.json 2>&1
TN_ATTN_DBG=gpurun_out/attn_ab2_dbg.txt python tools/attn_bench.py --reps 1 --runs 3 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_exec.py -q -m gpu -k "attention" > gpurun_out/attn_ab2_pytest.log 2>&1; echo rc=$? >> gpurun_out/attn_ab2_pytest.log
