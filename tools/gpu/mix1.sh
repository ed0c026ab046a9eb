timeout 300 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "attention_bwd" 2>&1 | grep -E "passed|failed|Error|error|assert" | head -20
timeout 120 python tools/attn_bwd_bench.py 2>&1 | tail -1
timeout 120 python tools/attn_bwd_bench.py --causal 0 --reps 3 2>&1 | tail -1
B="timeout 300 python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 3"
$B --exec-cfg '{"dependencies": "device"}' 2>&1 | tail -1 | grep -o '"exec_cfg.*\|"step_s": [^]]*]\|"frac_of_duplex_bound": [0-9.]*' | tr '\n' ' '; echo
$B --exec-cfg '{"dependencies": "device", "streams_per_device": 8}' 2>&1 | tail -1 | grep -o '"step_s": [^]]*]\|"frac_of_duplex_bound": [0-9.]*' | tr '\n' ' '; echo
$B --exec-cfg '{"dependencies": "device", "lookahead": 2}' 2>&1 | tail -1 | grep -o '"step_s": [^]]*]\|"frac_of_duplex_bound": [0-9.]*' | tr '\n' ' '; echo
$B 2>&1 | tail -1 | grep -o '"step_s": [^]]*]\|"frac_of_duplex_bound": [0-9.]*' | tr '\n' ' '; echo
