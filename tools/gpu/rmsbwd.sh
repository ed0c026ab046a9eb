timeout 600 python -m pytest tests/test_gpu_exec.py -q -m gpu -k "rmsnorm_bwd or training_rowops or lora" > gpurun_out/rmsbwd_pytest.log 2>&1; echo rc=$? >> gpurun_out/rmsbwd_pytest.log
PARITY_LOG=gpurun_out/parity_rms.jsonl timeout 600 python -m pytest tests/test_gpu_baseline_sizes.py -q -m gpu -k "config4" >> gpurun_out/rmsbwd_pytest.log 2>&1; echo rc=$? >> gpurun_out/rmsbwd_pytest.log
timeout 800 python tools/bench_lora.py --dump gpurun_out/lora_dump2.json > gpurun_out/lora_dump2.log 2>&1
