#!/bin/bash
# Builds abso/lib_prof.so: the library with attention.cu compiled -DTN_ATTN_PROF
# (per-block clock64 trace of the heaviest pair, printed by the kernel).
set -e
cd "$(dirname "$0")/../paper_2405_16283_b200/csrc"
JSONINC=$(python3 -c "import site,os;print([os.path.join(p,'include/cudnn_frontend/thirdparty') for p in site.getsitepackages()][0])")
nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xcompiler -fopenmp -isystem $JSONINC \
  --expt-relaxed-constexpr -DTN_ATTN_PROF -c kernels/attention.cu -o /tmp/attn_prof.o
objs=$(ls ../lib/obj/core/*.o ../lib/obj/*.o ../lib/obj/exec/*.o ../lib/obj/kernels/*.o | grep -v attention.cu.o)
mkdir -p ../../abso
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../abso/lib_prof.so $objs /tmp/attn_prof.o -Xcompiler -fopenmp -lgomp -cudart static -ldl -lpthread -lrt
