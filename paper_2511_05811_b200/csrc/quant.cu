// K0 amax and K1 two-level MOSS quantizer (row-wise + column-wise), plus the
// per-tensor encode used for weight copies.
//
// Reference semantics: quant_two_level (quantize.py:127-173),
// quant_per_tensor (quantize.py:92-98), _quantize_weight (train.py:113-118).
// HBM-bound: the quantizer's algorithmic traffic is 2 B (bf16 in) + 1 B codes
// + 1/32 B scale per element per orientation.
#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

// ------------------------------------------------------------------ K0 amax
// max |x| as f32 bits: abs-bits are ordered like the magnitudes, and any
// NaN/Inf lands >= 0x7F800000, so one integer max also detects non-finite input.
template <typename T>
__global__ void __launch_bounds__(256) amax_kernel(const T* __restrict__ x, int64_t n, float* amax,
                                                   uint32_t* flags) {
    const int64_t nvec = n / 8;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    uint32_t m = 0;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // back to front, 4 independent 8-element vectors in flight per thread
    for (; i + 3 * stride < nvec; i += 4 * stride) {
        float v[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) Vec8<T>::load(x + (nvec - 1 - (i + u * stride)) * 8, v[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) m = max(m, __float_as_uint(v[u][j]) & 0x7FFFFFFFu);
    }
    for (; i < nvec; i += stride) {
        float v[8];
        Vec8<T>::load(x + (nvec - 1 - i) * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) m = max(m, __float_as_uint(v[j]) & 0x7FFFFFFFu);
    }
    if (blockIdx.x == 0) {
        for (int64_t t = nvec * 8 + threadIdx.x; t < n; t += blockDim.x) {
            float f;
            if constexpr (sizeof(T) == 2) f = __bfloat162float(x[t]); else f = (float)x[t];
            m = max(m, __float_as_uint(f) & 0x7FFFFFFFu);
        }
    }
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    __shared__ uint32_t red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t r = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0u;
        r = __reduce_max_sync(0xFFFFFFFFu, r);
        if (threadIdx.x == 0) {
            if (r >= 0x7F800000u) atomicOr(flags, MOSS_FLAG_NONFINITE);
            else if (r) atomicMax(reinterpret_cast<uint32_t*>(amax), r);
        }
    }
}

// ------------------------------------------------------------------ K1 quantizer
// CTA tile: 32 rows x 256 columns, 256 threads.  Row pass straight from
// registers (4 lanes own one 32-element block); the column pass reads the
// tile back from shared memory (one thread per column, 32 rows = one block)
// and writes codes of x^T so the wgrad GEMM gets a K-major operand.
constexpr int QT_ROWS = 32;
constexpr int QT_COLS = 256;

template <typename T, bool ROW, bool COL>
__global__ void __launch_bounds__(256) quant_mx2_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                        const float* __restrict__ amax_p, uint8_t* codes,
                                                        uint8_t* sf, uint8_t* micro, uint8_t* codes_t,
                                                        uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                                                        uint32_t* flags) {
    __shared__ float tile[COL ? QT_ROWS : 1][QT_COLS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t c0 = (int64_t)blockIdx.x * QT_COLS;
    const int64_t r0 = (int64_t)blockIdx.y * QT_ROWS;
    const float amax = *amax_p;
    const float g = global_scale_from_amax(amax);
    if (g_out && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *g_out = g;
    bool rerr = false, bad = false;
    const int64_t nb_row = cols >> 5;
    const int64_t kch_row = (nb_row + 3) >> 2;

#pragma unroll
    for (int it = 0; it < QT_ROWS / 8; ++it) {
        const int lr = it * 8 + warp;
        const int64_t r = r0 + lr;
        const int64_t c = c0 + lane * 8;
        const bool valid = (r < rows) && (c < cols);
        float v[8];
        if (valid) {
            Vec8<T>::load(x + r * cols + c, v);
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f;
        }
        if (ROW) {
            float bm = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                bad |= nonfinite(v[j]);
                bm = fmaxf(bm, fabsf(v[j]));
            }
            bm = fmaxf(bm, __shfl_xor_sync(0xFFFFFFFFu, bm, 1));
            bm = fmaxf(bm, __shfl_xor_sync(0xFFFFFFFFu, bm, 2));
            float eff;
            const uint32_t code = block_scale(bm, g, eff, rerr);
            if (valid) {
                if (codes) {
                    uint2 pk;
                    pk.x = e4m3x4(__fdiv_rn(v[0], eff), __fdiv_rn(v[1], eff), __fdiv_rn(v[2], eff), __fdiv_rn(v[3], eff));
                    pk.y = e4m3x4(__fdiv_rn(v[4], eff), __fdiv_rn(v[5], eff), __fdiv_rn(v[6], eff), __fdiv_rn(v[7], eff));
                    *reinterpret_cast<uint2*>(codes + r * cols + c) = pk;
                }
                if ((lane & 3) == 0) {
                    const int64_t kb = c >> 5;
                    if (sf) sf[sf_offset(r, kb, kch_row)] = (uint8_t)code;
                    if (micro) micro[r * nb_row + kb] = (uint8_t)code;
                }
            }
        }
        if (COL) {
            float4* dst = reinterpret_cast<float4*>(&tile[lr][lane * 8]);
            dst[0] = make_float4(v[0], v[1], v[2], v[3]);
            dst[1] = make_float4(v[4], v[5], v[6], v[7]);
        }
    }

    if (COL) {
        __syncthreads();
        const int64_t col = c0 + tid;
        if (col < cols && r0 + QT_ROWS <= rows) {
            float bm = 0.f;
#pragma unroll
            for (int j = 0; j < QT_ROWS; ++j) {
                bad |= nonfinite(tile[j][tid]);
                bm = fmaxf(bm, fabsf(tile[j][tid]));
            }
            float eff;
            const uint32_t code = block_scale(bm, g, eff, rerr);
            if (codes_t) {
                uint32_t w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    w[q] = e4m3x4(__fdiv_rn(tile[4 * q][tid], eff), __fdiv_rn(tile[4 * q + 1][tid], eff),
                                  __fdiv_rn(tile[4 * q + 2][tid], eff), __fdiv_rn(tile[4 * q + 3][tid], eff));
                uint4* dst = reinterpret_cast<uint4*>(codes_t + col * rows + r0);
                dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
            const int64_t nb_t = rows >> 5;
            const int64_t kb = r0 >> 5;
            if (sf_t) sf_t[sf_offset(col, kb, (nb_t + 3) >> 2)] = (uint8_t)code;
            if (micro_t) micro_t[col * nb_t + kb] = (uint8_t)code;
        }
    }
    if (__any_sync(0xFFFFFFFFu, rerr) && lane == 0) atomicOr(flags, MOSS_FLAG_E8M0_RANGE);
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, MOSS_FLAG_NONFINITE);
}

// ------------------------------------------------------------------ K1 fast path (bf16)
// Persistent, TMA-fed: 32 x 256 bf16 tiles (16 KB) land in shared memory in
// the TMA 128B-swizzle layout through a QF_STAGES-deep mbarrier ring; each of
// the 256 threads then owns exactly one 32-element block in each pass (row
// pass: (row, k-block); column pass: one column of the 32-row block), so the
// per-block scale math runs once per block and every element costs one
// max, one exact block_div and half a cvt.  Non-finite inputs are detected
// by K0 (amax), not here.
constexpr int QF_ROWS = 32;
constexpr int QF_COLS = 256;
constexpr int QF_STAGES = 3;
constexpr int QF_TILE = QF_ROWS * QF_COLS * 2;

// byte offset of element (r, c) inside a tile: four 64-column TMA boxes of
// 32 rows x 128 B, 16 B chunks XOR-swizzled with the row (SWIZZLE_128B)
__device__ __forceinline__ uint32_t qf_off(int r, int c) {
    return (uint32_t)((c >> 6) * 4096 + r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4) + ((c & 7) << 1));
}

__device__ __forceinline__ void bf16x8(uint4 u, float* v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

template <bool ROW, bool COL>
__global__ void __launch_bounds__(256) quant_mx2_tma_kernel(const __grid_constant__ CUtensorMap tmx, int rows,
                                                            int cols, const float* __restrict__ amax_p,
                                                            uint8_t* codes, uint8_t* sf, uint8_t* micro,
                                                            uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                                                            float* g_out, uint32_t* flags) {
    extern __shared__ uint8_t qsmem_raw[];
    uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(qsmem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(tiles + QF_STAGES * QF_TILE);
    const int tid = threadIdx.x;
    const int ctiles = cols / QF_COLS;
    const int ntiles = ctiles * (rows / QF_ROWS);
    if (tid == 0) {
        for (int s = 0; s < QF_STAGES; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int tile, int s) {
        const int r0 = (tile / ctiles) * QF_ROWS, c0 = (tile % ctiles) * QF_COLS;
        mbar_arrive_expect_tx(&full[s], QF_TILE);
#pragma unroll
        for (int b = 0; b < 4; ++b) tma_load_2d(tiles + s * QF_TILE + b * 4096, &tmx, &full[s], c0 + b * 64, r0);
    };
    if (tid == 0) {
        for (int s = 0; s < QF_STAGES; ++s) {
            const int tile = blockIdx.x + s * gridDim.x;
            if (tile < ntiles) issue(tile, s);
        }
    }
    const float g = global_scale_from_amax(*amax_p);
    if (g_out && blockIdx.x == 0 && tid == 0) *g_out = g;
    const int nb_row = cols >> 5, kch_row = (nb_row + 3) >> 2;
    const int nb_t = rows >> 5, kch_t = (nb_t + 3) >> 2;
    bool rerr = false;
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it % QF_STAGES;
        mbar_wait(&full[s], (uint32_t)((it / QF_STAGES) & 1));
        const uint8_t* T = tiles + s * QF_TILE;
        const int r0 = (tile / ctiles) * QF_ROWS, c0 = (tile % ctiles) * QF_COLS;
        if (ROW) {
            const int r = tid & 31, kb = tid >> 5;
            float v[32];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                bf16x8(*reinterpret_cast<const uint4*>(T + qf_off(r, kb * 32 + q * 8)), v + 8 * q);
            float bm = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) bm = fmaxf(bm, fabsf(v[j]));
            float eff;
            const uint32_t code = block_scale(bm, g, eff, rerr);
            const BlockDiv d = make_block_div(eff);
            uint32_t w[8];
            encode_block32(v, d, w);
            const int64_t row = r0 + r;
            const int kbg = (c0 >> 5) + kb;
            if (codes) {
                uint4* dst = reinterpret_cast<uint4*>(codes + row * cols + c0 + kb * 32);
                dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
            if (sf) sf[sf_offset(row, kbg, kch_row)] = (uint8_t)code;
            if (micro) micro[row * nb_row + kbg] = (uint8_t)code;
        }
        if (COL) {
            const int c = tid;
            float v[32];
#pragma unroll
            for (int r = 0; r < 32; ++r)
                v[r] = __uint_as_float((uint32_t)(*reinterpret_cast<const uint16_t*>(T + qf_off(r, c))) << 16);
            float bm = 0.f;
#pragma unroll
            for (int j = 0; j < 32; ++j) bm = fmaxf(bm, fabsf(v[j]));
            float eff;
            const uint32_t code = block_scale(bm, g, eff, rerr);
            const BlockDiv d = make_block_div(eff);
            uint32_t w[8];
            encode_block32(v, d, w);
            const int64_t col = c0 + c;
            if (codes_t) {
                uint4* dst = reinterpret_cast<uint4*>(codes_t + col * rows + r0);
                dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
                dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
            }
            if (sf_t) sf_t[sf_offset(col, r0 >> 5, kch_t)] = (uint8_t)code;
            if (micro_t) micro_t[col * nb_t + (r0 >> 5)] = (uint8_t)code;
        }
        __syncthreads();  // every thread is done reading stage s
        if (tid == 0) {
            const int next = tile + QF_STAGES * gridDim.x;
            if (next < ntiles) issue(next, s);
        }
    }
    if (__any_sync(0xFFFFFFFFu, rerr) && (tid & 31) == 0) atomicOr(flags, MOSS_FLAG_E8M0_RANGE);
}

// ------------------------------------------------------------------ per-tensor encode
template <typename T>
__global__ void __launch_bounds__(256) encode_scaled_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                            const float* scale_p, float scale_host,
                                                            int from_amax, uint8_t* codes, uint8_t* codes_t,
                                                            float* scale_out, uint32_t* nsat, uint32_t* flags) {
    __shared__ __align__(16) uint8_t ctile[QT_ROWS][QT_COLS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t c0 = (int64_t)blockIdx.x * QT_COLS;
    const int64_t r0 = (int64_t)blockIdx.y * QT_ROWS;
    float scale = scale_host;
    if (scale_p) scale = from_amax ? global_scale_from_amax(*scale_p) : *scale_p;
    const float lim = __fmul_rn(scale, kE4M3Max);
    if (scale_out && blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *scale_out = scale;
    uint32_t sat = 0;
    bool bad = false;
#pragma unroll
    for (int it = 0; it < QT_ROWS / 8; ++it) {
        const int lr = it * 8 + warp;
        const int64_t r = r0 + lr;
        const int64_t c = c0 + lane * 8;
        uint2 pk = make_uint2(0, 0);
        if (r < rows && c < cols) {
            float v[8];
            Vec8<T>::load(x + r * cols + c, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                bad |= nonfinite(v[j]);
                sat += fabsf(v[j]) > lim;
            }
            pk.x = e4m3x4(__fdiv_rn(v[0], scale), __fdiv_rn(v[1], scale), __fdiv_rn(v[2], scale), __fdiv_rn(v[3], scale));
            pk.y = e4m3x4(__fdiv_rn(v[4], scale), __fdiv_rn(v[5], scale), __fdiv_rn(v[6], scale), __fdiv_rn(v[7], scale));
            if (codes) *reinterpret_cast<uint2*>(codes + r * cols + c) = pk;
        }
        if (codes_t) *reinterpret_cast<uint2*>(&ctile[lr][lane * 8]) = pk;
    }
    if (codes_t) {
        __syncthreads();
        const int64_t col = c0 + tid;
        if (col < cols && r0 + QT_ROWS <= rows) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q)
                w[q] = (uint32_t)ctile[4 * q][tid] | ((uint32_t)ctile[4 * q + 1][tid] << 8) |
                       ((uint32_t)ctile[4 * q + 2][tid] << 16) | ((uint32_t)ctile[4 * q + 3][tid] << 24);
            uint4* dst = reinterpret_cast<uint4*>(codes_t + col * rows + r0);
            dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
            dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
    }
    if (nsat) {
        sat = __reduce_add_sync(0xFFFFFFFFu, sat);
        if (lane == 0 && sat) atomicAdd(nsat, sat);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, MOSS_FLAG_NONFINITE);
}

// ------------------------------------------------------------------ launchers
int launch_amax(const void* x, int dtype, int64_t n, float* amax, uint32_t* flags, cudaStream_t st) {
    if (cudaMemsetAsync(amax, 0, sizeof(float), st) != cudaSuccess) return MOSS_ERR_CUDA;
    int64_t nvec = n / 8;
    int64_t want = (nvec + 255) / 256;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * 8));
    if (dtype == MOSS_BF16)
        amax_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, n, amax, flags);
    else
        amax_kernel<float><<<grid, 256, 0, st>>>((const float*)x, n, amax, flags);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

template <typename T>
static void launch_quant_t(const T* x, int64_t rows, int64_t cols, const float* amax, uint8_t* codes, uint8_t* sf,
                           uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                           uint32_t* flags, cudaStream_t st) {
    dim3 grid((unsigned)((cols + QT_COLS - 1) / QT_COLS), (unsigned)((rows + QT_ROWS - 1) / QT_ROWS));
    const bool row = codes || sf || micro;
    const bool col = codes_t || sf_t || micro_t;
    if (row && col)
        quant_mx2_kernel<T, true, true><<<grid, 256, 0, st>>>(x, rows, cols, amax, codes, sf, micro, codes_t, sf_t,
                                                              micro_t, g_out, flags);
    else if (col)
        quant_mx2_kernel<T, false, true><<<grid, 256, 0, st>>>(x, rows, cols, amax, codes, sf, micro, codes_t, sf_t,
                                                               micro_t, g_out, flags);
    else
        quant_mx2_kernel<T, true, false><<<grid, 256, 0, st>>>(x, rows, cols, amax, codes, sf, micro, codes_t, sf_t,
                                                               micro_t, g_out, flags);
}

static bool launch_quant_tma(const void* x, int64_t rows, int64_t cols, const float* amax, uint8_t* codes,
                             uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                             float* g_out, uint32_t* flags, cudaStream_t st) {
    if (rows % QF_ROWS || cols % QF_COLS || rows > INT32_MAX || cols > INT32_MAX) return false;
    CUtensorMap map;
    if (!make_tmap_2d(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, rows, cols, 64, QF_ROWS,
                      CU_TENSOR_MAP_SWIZZLE_128B))
        return false;
    const int smem = QF_STAGES * QF_TILE + 64 + 1024;
    const bool row = codes || sf || micro;
    const bool col = codes_t || sf_t || micro_t;
    auto kern = row && col ? quant_mx2_tma_kernel<true, true>
                           : (col ? quant_mx2_tma_kernel<false, true> : quant_mx2_tma_kernel<true, false>);
    static bool attr[3] = {false, false, false};
    const int ki = row && col ? 0 : (col ? 1 : 2);
    if (!attr[ki]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr[ki] = true;
    }
    const int64_t ntiles = (rows / QF_ROWS) * (cols / QF_COLS);
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count() * 4);
    kern<<<grid, 256, smem, st>>>(map, (int)rows, (int)cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out,
                                  flags);
    return true;
}

int launch_quant_mx2(const void* x, int dtype, int64_t rows, int64_t cols, const float* amax, uint8_t* codes,
                     uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                     uint32_t* flags, cudaStream_t st) {
    if (dtype == MOSS_BF16 &&
        launch_quant_tma(x, rows, cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out, flags, st))
        return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
    if (dtype == MOSS_BF16)
        launch_quant_t((const __nv_bfloat16*)x, rows, cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out,
                       flags, st);
    else
        launch_quant_t((const float*)x, rows, cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out, flags, st);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_encode_scaled(const void* x, int dtype, int64_t rows, int64_t cols, const float* scale, float scale_host,
                         int from_amax, uint8_t* codes, uint8_t* codes_t, float* scale_out, uint32_t* nsat,
                         uint32_t* flags, cudaStream_t st) {
    dim3 grid((unsigned)((cols + QT_COLS - 1) / QT_COLS), (unsigned)((rows + QT_ROWS - 1) / QT_ROWS));
    if (dtype == MOSS_BF16)
        encode_scaled_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, rows, cols, scale,
                                                                  scale_host, from_amax, codes, codes_t, scale_out, nsat, flags);
    else
        encode_scaled_kernel<float><<<grid, 256, 0, st>>>((const float*)x, rows, cols, scale, scale_host, from_amax,
                                                          codes, codes_t, scale_out, nsat, flags);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

}  // namespace moss
