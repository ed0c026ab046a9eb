python tools/gemm_bench.py --residual 4096x22016x64 4096x12288x64 4096x4096x64 4096x11008x64 4096x4096x4096 4096x4096x11008 2>&1 | grep "^{" | cut -c1-120 > gpurun_out/k64b.txt
python tools/gemm_bench.py --residual 4096x22016x64 4096x4096x4096 2>&1 | grep "^{" | cut -c1-120 >> gpurun_out/k64b.txt
timeout 600 python -m pytest tests/test_gpu_exec.py -q -m gpu -k "gemm" > gpurun_out/k64b_pytest.log 2>&1; echo rc=$? >> gpurun_out/k64b_pytest.log
