# config-4 overlap study: traced dump + plan/executor variants
timeout 600 python tools/bench_lora.py --steps 3 --dump gpurun_out/lora_dump.json 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --horizon greedy 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --exec-cfg '{"lookahead": 1}' 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --exec-cfg '{"dependencies": "device"}' 2>&1 | tail -1
timeout 600 python tools/bench_lora.py --steps 3 --cap-gib 20 2>&1 | tail -1
