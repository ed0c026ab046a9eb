timeout 900 python -m pytest tests/test_gpu_exec.py -m gpu -q -x -k "dispatch or residency or lora or offload or graph" 2>&1 | tail -1
timeout 300 python tools/trace_run.py --residency device --cfg '{"device_inputs": "copy"}' --tag value > /dev/null 2>&1
timeout 600 python tools/ab_exec_cfg.py '{"device_inputs": "copy"}' '{"device_inputs": "copy", "kernel_slots": true}' 2>&1 | tail -3
AB_RESIDENCY=host AB_REPS=4 timeout 600 python tools/ab_exec_cfg.py '{}' '{"kernel_slots": true}' 2>&1 | tail -3
