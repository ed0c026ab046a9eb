python tools/gemm_bench.py --residual 4096x22016x64 4096x12288x64 4096x4096x4096 4096x4096x11008 2>&1 | grep "^{" | cut -c1-100 > gpurun_out/pf_k.txt
timeout 600 python -m pytest tests/test_gpu_exec.py -q -m gpu -k "gemm" > gpurun_out/pf_k_pytest.log 2>&1; echo rc=$? >> gpurun_out/pf_k_pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel_2sm -s 0 -c 4 -o gpurun_out/r2g_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-offload-leg --no-other-configs --layers 2 > /dev/null 2>&1
for r in 1 2; do python bench.py --steps 10 --warmup 3 --no-offload-leg --no-other-configs --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], json.dumps({k:v['ms'] for k,v in d['roofline']['gemm_classes'].items()}))"; done >> gpurun_out/pf_k.txt 2>&1
