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
    if (zero_word(amax, st) != cudaSuccess) return MOSS_ERR_CUDA;
    int64_t nvec = n / 8;
    int64_t want = (nvec + 255) / 256;
    // one full wave: resident CTAs per SM x SMs (a partial second wave doubled the tail)
    static int occ[2] = {0, 0};
    const int di = dtype == MOSS_BF16;
    if (!occ[di]) {
        if (di)
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[di], amax_kernel<__nv_bfloat16>, 256, 0);
        else
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[di], amax_kernel<float>, 256, 0);
        if (occ[di] < 1) occ[di] = 4;
    }
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sm_count() * occ[di]));
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

bool launch_quant_v4(const void* x, int64_t rows, int64_t cols, float* amax, int amax_given, uint8_t* codes,
                     uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                     uint32_t* ws, uint32_t* flags, cudaStream_t st, int* status);

int launch_quant_mx2(const void* x, int dtype, int64_t rows, int64_t cols, const float* amax, uint8_t* codes,
                     uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                     uint32_t* flags, cudaStream_t st) {
    int status = MOSS_OK;
    // the TMA-tiled kernel in its given-amax mode (reads *amax, never writes it)
    if (dtype == MOSS_BF16 && launch_quant_v4(x, rows, cols, const_cast<float*>(amax), 1, codes, sf, micro, codes_t,
                                              sf_t, micro_t, g_out, nullptr, flags, st, &status))
        return status;
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

namespace moss {
// Single-launch quantizer (K0 folded into K1) where the v4 kernel covers the
// shape; otherwise K0 (unless the producer supplied amax) + K1.
int launch_quant_fused(const void* x, int dtype, int64_t rows, int64_t cols, float* amax, int amax_given,
                       uint8_t* codes, uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                       float* g_out, uint32_t* ws, uint32_t* flags, cudaStream_t st) {
    int status = MOSS_OK;
    if (dtype == MOSS_BF16 && launch_quant_v4(x, rows, cols, amax, amax_given, codes, sf, micro, codes_t, sf_t,
                                              micro_t, g_out, ws, flags, st, &status))
        return status;
    if (!amax_given) {
        status = launch_amax(x, dtype, rows * cols, amax, flags, st);
        if (status != MOSS_OK) return status;
    }
    return launch_quant_mx2(x, dtype, rows, cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out, flags, st);
}
}  // namespace moss
