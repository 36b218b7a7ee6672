// K3: AdamW fused with MOSS automatic weight scaling and the FP8 weight copy.
//
// One pass over the parameters: read W, G, m, v; write W', m', v' and the
// E4M3 codes of W' at the predicted scale s_{t+1} (and their transpose for
// the dgrad GEMM).  The scale itself advances on the host in O(1)
// (s_{t+1} = s_t + eta/448, autoscale.py:71-79) — no max-reduction here
// except the optional amax of W' that rescale steps (autoscale.py:86-96)
// and the dominance diagnostic (train.py:163-167) consume.
//
// Update rule (optim.py:78-106, computed in f32):
//   g  <- g + wd*w                  (coupled decay only)
//   m  <- b1 m + (1-b1) g ; v <- b2 v + (1-b2) g^2
//   d  = lr * (m/bc1) / (sqrt(v/bc2) + eps)
//   w' = w - d [- lr*wd*w  (decoupled)]
// Algorithmic traffic: 16 B read + 12 B written + 1 B code (+1 B transposed
// code) per parameter with f32 grads (29 / 30 B).
#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

template <typename G> struct GradLoad;
template <> struct GradLoad<float> {
    __device__ __forceinline__ static void load(const float* p, float (&v)[8]) { Vec8<float>::load(p, v); }
};
template <> struct GradLoad<__nv_bfloat16> {
    __device__ __forceinline__ static void load(const __nv_bfloat16* p, float (&v)[8]) {
        Vec8<__nv_bfloat16>::load(p, v);
    }
};

__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

constexpr int AT_ROWS = 32;
constexpr int AT_COLS = 256;

template <typename GT, bool ENC, bool TRANS>
__global__ void __launch_bounds__(256) adamw_fp8_kernel(float* __restrict__ w, const GT* __restrict__ g,
                                                        float* __restrict__ m, float* __restrict__ v, int64_t rows,
                                                        int64_t cols, moss_adam_params p, float enc_scale,
                                                        const moss_adam_params* __restrict__ p_dev,
                                                        const float* __restrict__ enc_dev, float* scale_out,
                                                        uint8_t* __restrict__ w_fp8, uint8_t* __restrict__ w_fp8_t,
                                                        float* w_amax, uint32_t* nsat, uint32_t* flags) {
    // device-resident hyper-parameters (CUDA-graph replays): read them once per CTA
    if (p_dev) p = *p_dev;
    if (enc_dev) enc_scale = *enc_dev;
    // error gate: an earlier kernel of this step flagged a non-finite / out-of-range
    // value -> no update at all (the reference raises before mutating, optim.py:89-90)
    if (*reinterpret_cast<volatile uint32_t*>(flags) & MOSS_FLAG_SKIP_MASK) {
        if (p.step && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) atomicMin(flags + 1, p.step);
        return;
    }
    if (scale_out && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) *scale_out = enc_scale;
    __shared__ __align__(16) uint8_t ctile[TRANS ? AT_ROWS : 1][AT_COLS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t c0 = (int64_t)blockIdx.x * AT_COLS;
    const int64_t r0 = (int64_t)blockIdx.y * AT_ROWS;
    const float lim = __fmul_rn(enc_scale, kE4M3Max);
    const float om1 = 1.0f - p.beta1, om2 = 1.0f - p.beta2;
    const float decay = p.lr * p.weight_decay;
    // bias corrections as multiplies, sqrt/division by the SFU: the update is
    // held to a tolerance vs the float64 reference (|dW| <= 1e-3 eta per step,
    // SURVEY.md 8(c)); only the FP8 encode below must be IEEE-exact.
    const float ibc1 = 1.0f / p.bc1, ibc2 = 1.0f / p.bc2;
    uint32_t amax_bits = 0, sat = 0;
    bool bad = false;
    const int64_t c = c0 + lane * 8;
    const bool col_ok = c < cols;
    // one row of look-ahead: the next row's four vectors are in flight while this row computes
    float wv[8], gv[8], mv[8], vv[8];
    auto load_row = [&](int it, float (&W)[8], float (&Gd)[8], float (&M)[8], float (&V)[8]) {
        const int64_t r = r0 + it * 8 + warp;
        if (r < rows && col_ok) {
            const int64_t off = r * cols + c;
            Vec8<float>::load(w + off, W);
            GradLoad<GT>::load(g + off, Gd);
            Vec8<float>::load(m + off, M);
            Vec8<float>::load(v + off, V);
        }
    };
    load_row(0, wv, gv, mv, vv);
#pragma unroll
    for (int it = 0; it < AT_ROWS / 8; ++it) {
        const int lr = it * 8 + warp;
        const int64_t r = r0 + lr;
        float wn_[8], gn_[8], mn_[8], vn_[8];
        if (it + 1 < AT_ROWS / 8) load_row(it + 1, wn_, gn_, mn_, vn_);
        uint2 pk = make_uint2(0, 0);
        if (r < rows && col_ok) {
            const int64_t off = r * cols + c;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float gj = gv[j] * p.grad_scale;
                if (nonfinite(gj)) {  // leave this element untouched; host raises
                    bad = true;
                    continue;
                }
                if (!p.decoupled) gj = fmaf(p.weight_decay, wv[j], gj);
                mv[j] = fmaf(p.beta1, mv[j], om1 * gj);
                vv[j] = fmaf(p.beta2, vv[j], om2 * gj * gj);
                float sq;
                asm("sqrt.approx.f32 %0, %1;" : "=f"(sq) : "f"(vv[j] * ibc2));
                const float delta = __fdividef(p.lr * (mv[j] * ibc1), sq + p.eps);
                float wn = wv[j] - delta;
                if (p.decoupled) wn = fmaf(-decay, wv[j], wn);
                wv[j] = wn;
            }
            store8(w + off, wv);
            store8(m + off, mv);
            store8(v + off, vv);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                amax_bits = max(amax_bits, __float_as_uint(wv[j]) & 0x7FFFFFFFu);
                sat += fabsf(wv[j]) > lim;
            }
            if (ENC) {
                pk.x = e4m3x4(__fdiv_rn(wv[0], enc_scale), __fdiv_rn(wv[1], enc_scale), __fdiv_rn(wv[2], enc_scale),
                              __fdiv_rn(wv[3], enc_scale));
                pk.y = e4m3x4(__fdiv_rn(wv[4], enc_scale), __fdiv_rn(wv[5], enc_scale), __fdiv_rn(wv[6], enc_scale),
                              __fdiv_rn(wv[7], enc_scale));
                if (w_fp8) *reinterpret_cast<uint2*>(w_fp8 + off) = pk;
            }
        }
        if (TRANS) *reinterpret_cast<uint2*>(&ctile[lr][lane * 8]) = pk;
        if (it + 1 < AT_ROWS / 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                wv[j] = wn_[j]; gv[j] = gn_[j]; mv[j] = mn_[j]; vv[j] = vn_[j];
            }
        }
    }
    if (TRANS) {
        __syncthreads();
        const int64_t col = c0 + tid;
        if (col < cols && r0 + AT_ROWS <= rows) {
            uint32_t q[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                q[k] = (uint32_t)ctile[4 * k][tid] | ((uint32_t)ctile[4 * k + 1][tid] << 8) |
                       ((uint32_t)ctile[4 * k + 2][tid] << 16) | ((uint32_t)ctile[4 * k + 3][tid] << 24);
            uint4* dst = reinterpret_cast<uint4*>(w_fp8_t + col * rows + r0);
            dst[0] = make_uint4(q[0], q[1], q[2], q[3]);
            dst[1] = make_uint4(q[4], q[5], q[6], q[7]);
        }
    }
    if (w_amax) {
        amax_bits = __reduce_max_sync(0xFFFFFFFFu, amax_bits);
        if (lane == 0 && amax_bits) atomicMax(reinterpret_cast<uint32_t*>(w_amax), amax_bits);
    }
    if (nsat) {
        sat = __reduce_add_sync(0xFFFFFFFFu, sat);
        if (lane == 0 && sat) atomicAdd(nsat, sat);
    }
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, MOSS_FLAG_GRAD_NONFINITE);
}

template <typename T>
__global__ void __launch_bounds__(256) check_finite_kernel(const T* __restrict__ x, int64_t n, uint32_t bit,
                                                           uint32_t* flags) {
    bool bad = false;
    const int64_t n8 = n / 8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
        float v[8];
        Vec8<T>::load(x + i * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) bad |= nonfinite(v[j]);
    }
    for (int64_t i = n8 * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= nonfinite(static_cast<float>(x[i]));
    if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, bit);
}

int launch_check_finite(const void* x, int dtype, int64_t n, uint32_t bit, uint32_t* flags, cudaStream_t st) {
    if (n <= 0) return MOSS_OK;
    const int64_t want = (n / 8 + 255) / 256;
    const int grid = (int)std::min<int64_t>(std::max<int64_t>(want, 1), 148 * 8);
    if (dtype == MOSS_BF16)
        check_finite_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, n, bit, flags);
    else
        check_finite_kernel<float><<<grid, 256, 0, st>>>((const float*)x, n, bit, flags);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

template <typename GT>
static void launch_adamw_t(float* w, const GT* g, float* m, float* v, int64_t rows, int64_t cols,
                           const moss_adam_params& p, float enc_scale, const moss_adam_params* p_dev,
                           const float* enc_dev, float* scale_out, uint8_t* w_fp8, uint8_t* w_fp8_t,
                           float* w_amax, uint32_t* nsat, uint32_t* flags, cudaStream_t st) {
    dim3 grid((unsigned)((cols + AT_COLS - 1) / AT_COLS), (unsigned)((rows + AT_ROWS - 1) / AT_ROWS));
    if (w_fp8_t)
        adamw_fp8_kernel<GT, true, true><<<grid, 256, 0, st>>>(w, g, m, v, rows, cols, p, enc_scale, p_dev, enc_dev,
                                                               scale_out, w_fp8, w_fp8_t, w_amax, nsat, flags);
    else if (w_fp8)
        adamw_fp8_kernel<GT, true, false><<<grid, 256, 0, st>>>(w, g, m, v, rows, cols, p, enc_scale, p_dev, enc_dev,
                                                                scale_out, w_fp8, w_fp8_t, w_amax, nsat, flags);
    else
        adamw_fp8_kernel<GT, false, false><<<grid, 256, 0, st>>>(w, g, m, v, rows, cols, p, enc_scale, p_dev, enc_dev,
                                                                 scale_out, w_fp8, w_fp8_t, w_amax, nsat, flags);
}

int launch_adamw(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                 const moss_adam_params& p, float enc_scale, const moss_adam_params* p_dev, const float* enc_dev,
                 float* scale_out, uint8_t* w_fp8, uint8_t* w_fp8_t, float* w_amax, uint32_t* nsat,
                 uint32_t* flags, cudaStream_t st) {
    if (w_amax && zero_word(w_amax, st) != cudaSuccess) return MOSS_ERR_CUDA;
    if (g_dtype == MOSS_BF16)
        launch_adamw_t(w, (const __nv_bfloat16*)g, m, v, rows, cols, p, enc_scale, p_dev, enc_dev, scale_out, w_fp8,
                       w_fp8_t, w_amax, nsat, flags, st);
    else
        launch_adamw_t(w, (const float*)g, m, v, rows, cols, p, enc_scale, p_dev, enc_dev, scale_out, w_fp8, w_fp8_t,
                       w_amax, nsat, flags, st);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

}  // namespace moss
