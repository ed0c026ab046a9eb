python -m pytest tests/test_gpu_exec.py -m gpu -q -k "lora or unaligned or graph_mode or split_k or gemm_parity or dispatch_order or blockwise" 2>&1 | grep -E "^E  |FAILED|passed|failed" | head -20
A="--heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 3"
python tools/bench_longctx.py $A
python tools/bench_longctx.py $A --exec-cfg '{"dependencies": "device"}' --dump gpurun_out/lc_trace_dd.json
python tools/bench_longctx.py $A --exec-cfg '{"dependencies": "device", "lookahead": 3}'
python tools/bench_lora.py 2>&1 | tail -1
python tools/bench_lora.py --exec-cfg '{"dependencies": "device"}' 2>&1 | tail -1
python tools/bench_lora.py --exec-cfg '{"dependencies": "device", "lookahead": 3}' 2>&1 | tail -1
