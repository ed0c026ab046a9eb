// Probe: does programmatic dependent launch still overlap a kernel's launch
// with its predecessor when cudaEventRecord calls sit between them?
// Each kernel spins ~T us; B records globaltimer at entry (before
// griddepcontrol.wait) and after the wait. Prints B_entry - A_end.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__global__ void kA(unsigned long long* ts, int spin_us) {
    asm volatile("griddepcontrol.launch_dependents;");
    unsigned long long t0 = gt();
    while (gt() - t0 < spin_us * 1000ull) {}
    __syncthreads();
    if (threadIdx.x == 0) atomicMax(ts + 0, gt());  // A end (max over CTAs)
}
__global__ void kB(unsigned long long* ts) {
    unsigned long long e = gt();
    if (threadIdx.x == 0) atomicMin(ts + 1, e);  // B first entry
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicMin(ts + 2, gt());  // B after wait
}
int main() {
    unsigned long long* ts; cudaMalloc(&ts, 24);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t e1, e2, n1, n2;
    cudaEventCreate(&e1); cudaEventCreate(&e2);
    cudaEventCreateWithFlags(&n1, cudaEventDisableTiming); cudaEventCreateWithFlags(&n2, cudaEventDisableTiming);
    for (int mode = 0; mode < 12; ++mode) {  // bit0: PDL; bits1-3: 0 none, 1 two timing events, 2 two non-timing, 3 one timing, 4 one non-timing
        unsigned long long init[3] = {0, ~0ull, ~0ull};
        for (int rep = 0; rep < 3; ++rep) {
            cudaMemcpy(ts, init, 24, cudaMemcpyHostToDevice);
            kA<<<148, 128, 0, s>>>(ts, 50);
            const int ev = mode >> 1;
            if (ev == 1) { cudaEventRecord(e1, s); cudaEventRecord(e2, s); }
            if (ev == 2) { cudaEventRecord(n1, s); cudaEventRecord(n2, s); }
            if (ev == 3) { cudaEventRecord(e1, s); }
            if (ev == 4) { cudaEventRecord(n1, s); }
            if (ev == 5) { cudaEventRecord(n1, s); cudaEventRecord(e2, s); }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = 148; cfg.blockDim = 128; cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = (mode & 1);
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, kB, ts);
            cudaStreamSynchronize(s);
        }
        unsigned long long h[3]; cudaMemcpy(h, ts, 24, cudaMemcpyDeviceToHost);
        const char* names[] = {"none", "2 timing", "2 non-timing", "1 timing", "1 non-timing", "non-timing+timing"};
        printf("pdl=%d events=%-18s B_entry - A_end = %+.2f us, B_after_wait - A_end = %+.2f us (%s)\n", mode & 1,
               names[mode >> 1], ((long long)(h[1] - h[0])) / 1e3, ((long long)(h[2] - h[0])) / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
}
