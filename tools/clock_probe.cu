// Diagnostic (not product code): SM clock at a point in a stream.  One warp
// spins ~ns nanoseconds on %globaltimer and records the clock64 cycles it saw:
// MHz = cycles / ns * 1e3.  Built by tools/quant_clock_probe.py:
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o tools/_clock_probe.so tools/clock_probe.cu
#include <cstdint>
#include <cuda_runtime.h>

__global__ void clock_probe_kernel(unsigned long long* out, int slot, int ns) {
    uint64_t t0, t, c0, c1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    c0 = clock64();
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < (uint64_t)ns);
    c1 = clock64();
    if (threadIdx.x == 0) {
        out[2 * slot] = c1 - c0;
        out[2 * slot + 1] = t - t0;
    }
}

extern "C" int clock_probe(void* out, int slot, int ns, void* stream) {
    clock_probe_kernel<<<1, 32, 0, (cudaStream_t)stream>>>((unsigned long long*)out, slot, ns);
    return (int)cudaGetLastError();
}
