// Host-side helpers shared by the launchers: TMA tensor-map encoding through
// the driver entry point (no -lcuda link), SM count.
#pragma once
#include <cstdlib>

#include <cuda.h>
#include <cuda_runtime.h>

namespace moss {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn get_encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// 2-D row-major tensor [rows, cols] of `dtype`, box {box_cols, box_rows}.
inline bool make_tmap_2d(CUtensorMap* map, CUtensorMapDataType dtype, size_t elem_bytes, const void* ptr,
                         int64_t rows, int64_t cols, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
    EncodeTiledFn enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)(cols * elem_bytes)};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1u, 1u};
    return enc(map, dtype, 2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Launcher state that the CUDA runtime keeps per device (the shared-memory
// opt-in of cudaFuncSetAttribute, occupancy, SM count) is cached per device:
// one process may drive several GPUs.  (Occupancy of kernels without a
// dynamic shared-memory opt-in depends only on the kernel and the arch; those
// caches stay per process on this one-arch (sm_100a) build.)
constexpr int kMaxDevices = 64;

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return (dev >= 0 && dev < kMaxDevices) ? dev : 0;
}

inline int sm_count() {
    static int n[kMaxDevices] = {};
    const int dev = current_device();
    if (!n[dev]) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        n[dev] = v > 0 ? v : 148;
    }
    return n[dev];
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device);
// `done` is the caller's per-kernel static table
template <typename K>
inline bool smem_optin(K kern, int bytes, bool (&done)[kMaxDevices]) {
    const int dev = current_device();
    if (done[dev]) return true;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
    done[dev] = true;
    return true;
}

// Zero one 32-bit word on a stream.  A one-thread kernel rather than
// cudaMemsetAsync: inside a CUDA graph a memset node between two kernel nodes
// costs several microseconds of idle SMs on each side (kernel -> kernel
// transitions ~0.4 us).  MOSS_MEMSET_NODE=1 restores cudaMemsetAsync (A/B).
static __global__ void zero_word_kernel(uint32_t* p) { *p = 0u; }
inline bool memset_nodes() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_MEMSET_NODE");
        v = e ? (e[0] != '0') : 0;
    }
    return v != 0;
}
inline cudaError_t zero_word(void* p, cudaStream_t st) {
    if (memset_nodes()) return cudaMemsetAsync(p, 0, 4, st);
    zero_word_kernel<<<1, 1, 0, st>>>(reinterpret_cast<uint32_t*>(p));
    return cudaGetLastError();
}

}  // namespace moss
