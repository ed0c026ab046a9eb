# config 5 (64k blockwise, greedy lag 1, 6 GiB): executor variants with the plan-order default
B="timeout 300 python tools/bench_longctx.py --heads 8 --lag 1 --cap-gib 6 --horizon greedy --steps 3"
$B 2>&1 | tail -1 | cut -c1-420
$B --exec-cfg '{"streams_per_device": 8}' 2>&1 | tail -1 | cut -c1-420
$B --exec-cfg '{"dependencies": "device"}' 2>&1 | tail -1 | cut -c1-420
$B --exec-cfg '{"lookahead": 2}' 2>&1 | tail -1 | cut -c1-420
$B --exec-cfg '{"kernel_slots": false}' 2>&1 | tail -1 | cut -c1-420
$B --dump gpurun_out/c5_dump.json 2>&1 | tail -1 | cut -c1-100
