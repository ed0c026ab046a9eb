for t in auto narrow wide; do TN_GEMM_TILE=$t python tools/gemm_bench.py --residual 4096x22016x64 4096x4096x64 2>&1 | grep "^{" | cut -c1-120 | sed "s/^/$t /"; done > gpurun_out/k64.txt
for t in auto narrow wide; do TN_GEMM_TILE=$t python tools/gemm_bench.py 4096x22016x64 2>&1 | grep "^{" | cut -c1-120 | sed "s/^/noresid $t /"; done >> gpurun_out/k64.txt
timeout 300 ncu --set full --import-source on --clock-control none -k regex:gemm_kernel -c 1 -o gpurun_out/k64 python tools/gemm_bench.py --residual 4096x22016x64 > /dev/null 2>&1
