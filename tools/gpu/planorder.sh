# "plan-order" tie break vs fifo: config 4 (LoRA), config 5 (blockwise), dispatch-order tests
timeout 600 python -m pytest tests/test_gpu_exec.py -m gpu -q -k "dispatch or order or device_resid" 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --exec-cfg '{"tie_break": "plan-order"}' --dump gpurun_out/lora_dump_po.json 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --exec-cfg '{"tie_break": "plan-order"}' --compare 2>&1 | tail -1
timeout 600 python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 3 2>&1 | tail -1
timeout 600 python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 3 --exec-cfg '{"tie_break": "plan-order"}' 2>&1 | tail -1
