// Diagnostic microbenchmark (not product code): DRAM bandwidth of a pure
// 2-D TMA tile copy (bf16 [M, N] -> [M, N]) as a function of the tile shape,
// with the K1 quantizer's pipeline (persistent CTAs, a ring of smem slots,
// TMA load -> mbarrier -> TMA store from the same slot -> refill once read).
// Question answered: is the tiled access pattern itself the K1 ceiling?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_tile_copy tools/tma_tile_copy.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const CUtensorMap* m, uint64_t* bar, int c, int r) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(m), "r"(smem_u32(bar)), "r"(c), "r"(r)
        : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap* m, const void* src, int c, int r) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(m),
                 "r"(smem_u32(src)), "r"(c), "r"(r)
                 : "memory");
}

constexpr int SLOTS = 3;

// tile = R rows x (64 * NB) bf16 columns: NB boxes of 64 columns (128 B rows, SWIZZLE_128B)
__global__ void __launch_bounds__(128) tile_copy(const __grid_constant__ CUtensorMap src,
                                                 const __grid_constant__ CUtensorMap dst, int M, int N, int R, int NB) {
    extern __shared__ uint8_t raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    const int tile_bytes = R * NB * 128;
    uint64_t* full = reinterpret_cast<uint64_t*>(base + SLOTS * tile_bytes);
    const int ctiles = N / (64 * NB), ntiles = ctiles * (M / R);
    const int G = gridDim.x, b = blockIdx.x;
    const int n = ntiles > b ? (ntiles - b + G - 1) / G : 0;
    if (threadIdx.x != 0) return;   // one thread drives the whole pipeline
    for (int s = 0; s < SLOTS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    auto load = [&](int j) {
        const int t = b + j * G, s = j % SLOTS;
        const int r0 = (t / ctiles) * R, c0 = (t % ctiles) * 64 * NB;
        mbar_expect(&full[s], tile_bytes);
        for (int k = 0; k < NB; ++k) tma_load(base + s * tile_bytes + k * R * 128, &src, &full[s], c0 + 64 * k, r0);
    };
    for (int j = 0; j < n && j < SLOTS; ++j) load(j);
    uint32_t par = 0;
    for (int p = 0; p < n; ++p) {
        const int s = p % SLOTS;
        mbar_wait(&full[s], (par >> s) & 1u);
        par ^= 1u << s;
        const int t = b + p * G;
        const int r0 = (t / ctiles) * R, c0 = (t % ctiles) * 64 * NB;
        for (int k = 0; k < NB; ++k) tma_store(&dst, base + s * tile_bytes + k * R * 128, c0 + 64 * k, r0);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (p >= 1) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            if (p - 1 + SLOTS < n) load(p - 1 + SLOTS);
        }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int M = 8192, N = 22016 - 22016 % 1024 + 1024;   // 8192 x 22528 bf16 (369 MB each way)
    void *src, *dst;
    CK(cudaMalloc(&src, (size_t)M * N * 2));
    CK(cudaMalloc(&dst, (size_t)M * N * 2));
    CK(cudaMemset(src, 1, (size_t)M * N * 2));
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // torch-like linear copy reference
    for (int i = 0; i < 3; ++i) CK(cudaMemcpyAsync(dst, src, (size_t)M * N * 2, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(e0));
    for (int i = 0; i < 10; ++i) CK(cudaMemcpyAsync(dst, src, (size_t)M * N * 2, cudaMemcpyDeviceToDevice));
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf("cudaMemcpy D2D: %.0f GB/s\n", 2.0 * M * N * 2 * 10 / (ms * 1e6));
    const int shapes[][2] = {{256, 1}, {128, 1}, {128, 2}, {64, 4}, {32, 8}, {16, 16}, {64, 2}, {32, 4}};
    for (auto& sh : shapes) {
        const int R = sh[0], NB = sh[1];
        CUtensorMap ms_, md_;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)N * 2};
        cuuint32_t box[2] = {64u, (cuuint32_t)R};
        cuuint32_t es[2] = {1u, 1u};
        if (enc(&ms_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ||
            enc(&md_, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dst, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)) {
            printf("encode failed\n");
            return 1;
        }
        const int tile_bytes = R * NB * 128;
        const int smem = SLOTS * tile_bytes + 64 + 1024;
        CK(cudaFuncSetAttribute(tile_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, tile_copy, 128, smem));
        const int grid = sms * occ;
        for (int i = 0; i < 3; ++i) tile_copy<<<grid, 128, smem>>>(ms_, md_, M, N, R, NB);
        CK(cudaGetLastError());
        CK(cudaEventRecord(e0));
        for (int i = 0; i < 10; ++i) tile_copy<<<grid, 128, smem>>>(ms_, md_, M, N, R, NB);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms, e0, e1));
        printf("tile %3d x %4d (%2d KB, %d CTAs/SM x %d slots): %.0f GB/s\n", R, 64 * NB, tile_bytes / 1024, occ, SLOTS,
               2.0 * M * N * 2 * 10 / (ms * 1e6));
    }
    return 0;
}
