// Producer kernels of the MOSS activations and gradients (SURVEY.md 8(f)
// rank 1: producer-fused amax).
//
// In the Llama decoder every FP8 linear's input and output-gradient is made
// by one of these kernels: RMSNorm (forward: the qkv / gate_up inputs;
// backward: the o / down output-gradients), SwiGLU (forward: the down input;
// backward: the gate_up output-gradient) and RoPE (backward: the qkv
// output-gradient).  Each kernel writes its bf16 output AND max|output| —
// the tensor amax the two-level quantizer needs for g = amax/448
// (quantize.py:149-155) — so the quantizer runs in its producer-amax mode:
// one read of the tensor, no reduction pass, no grid barrier.
//
// The kernels are plain HBM-streaming elementwise / row-reduction kernels:
// 16-byte vector loads/stores, f32 arithmetic, one pass.  amax is reduced
// per CTA and merged with one atomicMax on the f32 bits (|y| >= 0 orders
// like its bits; NaN/Inf land above 0x7F800000 and the quantizer flags them).
// The caller zeroes the amax word (stream-ordered memset in the launcher).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

__device__ __forceinline__ void bf16x8_load(const __nv_bfloat16* p, float (&v)[8]) { Vec8<__nv_bfloat16>::load(p, v); }

__device__ __forceinline__ void unpack_bf16x8(const uint4& u, float (&v)[8]) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}

__device__ __forceinline__ uint4 bf16x8_pack(const float (&v)[8]) {
    uint4 o;
    o.x = pack_bf16(v[0], v[1]);
    o.y = pack_bf16(v[2], v[3]);
    o.z = pack_bf16(v[4], v[5]);
    o.w = pack_bf16(v[6], v[7]);
    return o;
}

// |v| of the bf16-ROUNDED values (the tensor the quantizer will read)
__device__ __forceinline__ uint32_t absmax_bits_bf16(const uint4& o) {
    const uint32_t a = __vmaxu2(o.x & 0x7FFF7FFFu, o.y & 0x7FFF7FFFu);
    const uint32_t b = __vmaxu2(o.z & 0x7FFF7FFFu, o.w & 0x7FFF7FFFu);
    const uint32_t c = __vmaxu2(a, b);
    return max(c & 0xFFFFu, c >> 16) << 16;   // as f32 bits
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 16);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 8);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    constexpr int NW = NT / 32;
    if (NW == 1) return v;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();   // red reuse across calls
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) s += red[i];
    return s;
}

__device__ __forceinline__ void block_amax_commit(uint32_t m, uint32_t* red_u, uint32_t* amax) {
    if (!amax) return;
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();
    if (lane == 0) red_u[warp] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) r = max(r, red_u[i]);
        if (r) atomicMax(amax, r);
    }
}

// ------------------------------------------------------------------ RMSNorm
// forward, one row per CTA iteration, NT threads x 8 elements (d = 8*NT):
//   x' = x + delta (bf16, when delta != null; written to x_out)
//   y  = bf16( f32(x') * rsqrt(mean(f32(x')^2) + eps) * w )
//   rstd[t] = rsqrt(...), amax = max |y|
template <int NT>
__global__ void __launch_bounds__(NT, (1024 / NT > 0 ? 1024 / NT : 1)) rmsnorm_fwd_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const __nv_bfloat16* __restrict__ delta,
                                                         __nv_bfloat16* __restrict__ x_out, const float* __restrict__ w,
                                                         float eps, __nv_bfloat16* __restrict__ y,
                                                         float* __restrict__ rstd, uint32_t* amax, int T, int d) {
    __shared__ float red[NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    const int c = threadIdx.x * 8;
    const bool act = c < d;
    float wv[8];
    if (act) {
        const float4 a = *reinterpret_cast<const float4*>(w + c);
        const float4 b = *reinterpret_cast<const float4*>(w + c + 4);
        wv[0] = a.x; wv[1] = a.y; wv[2] = a.z; wv[3] = a.w; wv[4] = b.x; wv[5] = b.y; wv[6] = b.z; wv[7] = b.w;
    }
    uint32_t m = 0;
    // one row of look-ahead: the next row's loads are in flight during this row's reduction
    uint4 xa = make_uint4(0, 0, 0, 0), da = make_uint4(0, 0, 0, 0);
    auto load = [&](int t, uint4& xr, uint4& dr) {
        if (act && t < T) {
            const int64_t off = (int64_t)t * d + c;
            xr = *reinterpret_cast<const uint4*>(x + off);
            if (delta) dr = *reinterpret_cast<const uint4*>(delta + off);
        }
    };
    load(blockIdx.x, xa, da);
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int64_t off = (int64_t)t * d + c;
        uint4 xn = make_uint4(0, 0, 0, 0), dn = make_uint4(0, 0, 0, 0);
        load(t + gridDim.x, xn, dn);
        float v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        float ss = 0.f;
        if (act) {
            unpack_bf16x8(xa, v);
            if (delta) {
                float dv[8];
                unpack_bf16x8(da, dv);
#pragma unroll
                for (int i = 0; i < 8; ++i) v[i] = __bfloat162float(__float2bfloat16_rn(v[i] + dv[i]));
                *reinterpret_cast<uint4*>(x_out + off) = bf16x8_pack(v);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) ss = fmaf(v[i], v[i], ss);
        }
        ss = block_sum<NT>(ss, red);
        const float r = rsqrtf(ss / (float)d + eps);
        if (threadIdx.x == 0) rstd[t] = r;
        if (act) {
            float o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = v[i] * r * wv[i];
            const uint4 ob = bf16x8_pack(o);
            *reinterpret_cast<uint4*>(y + off) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
        xa = xn;
        da = dn;
    }
    block_amax_commit(m, red_u, amax);
}

// The same forward with ONE WARP PER ROW (d = 256 * VPL, VPL <= 16): no block
// barriers, the whole row (and delta) in flight per warp — 16 KB per warp,
// 128 KB per SM — instead of one 8 KB row per 512-thread CTA between two
// __syncthreads.  Used for d % 256 == 0 (every Llama width here).
template <int VPL>
__global__ void __launch_bounds__(256) rmsnorm_fwd_warp_kernel(const __nv_bfloat16* __restrict__ x,
                                                               const __nv_bfloat16* __restrict__ delta,
                                                               __nv_bfloat16* __restrict__ x_out,
                                                               const float* __restrict__ w, float eps,
                                                               __nv_bfloat16* __restrict__ y, float* __restrict__ rstd,
                                                               uint32_t* amax, int T, int d) {
    __shared__ uint32_t red_u[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t m = 0;
    for (int t = blockIdx.x * 8 + warp; t < T; t += gridDim.x * 8) {
        const int64_t row = (int64_t)t * d;
        uint4 v[VPL];
#pragma unroll
        for (int i = 0; i < VPL; ++i) v[i] = *reinterpret_cast<const uint4*>(x + row + (i * 32 + lane) * 8);
        if (delta) {
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const uint4 dd = *reinterpret_cast<const uint4*>(delta + row + (i * 32 + lane) * 8);
                float a[8], b[8];
                unpack_bf16x8(v[i], a);
                unpack_bf16x8(dd, b);
#pragma unroll
                for (int j = 0; j < 8; ++j) a[j] += b[j];
                v[i] = bf16x8_pack(a);
                *reinterpret_cast<uint4*>(x_out + row + (i * 32 + lane) * 8) = v[i];
            }
        }
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            float a[8];
            unpack_bf16x8(v[i], a);
#pragma unroll
            for (int j = 0; j < 8; ++j) ss = fmaf(a[j], a[j], ss);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xFFFFFFFFu, ss, o);
        const float r = rsqrtf(ss / (float)d + eps);
        if (lane == 0) rstd[t] = r;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            const int c = (i * 32 + lane) * 8;
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float a[8];
            unpack_bf16x8(v[i], a);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] * r * wv[j];
            const uint4 ob = bf16x8_pack(a);
            *reinterpret_cast<uint4*>(y + row + c) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    block_amax_commit(m, red_u, amax);
}

// ---- v2 (d % 1024 == 0, i.e. the 7B width 4096): a CTA of NT = d/32 threads
// owns one row per iteration, each thread VPT = 4 strided 16-byte vectors
// (32 elements: consecutive threads read consecutive 16 B, fully coalesced).
// All of a row's loads (x and delta, or dy, x and d_res) are issued before any
// math; ~4-5 CTAs per SM keep 100+ KB in flight per SM.  One __syncthreads per
// row (the partial sums are double-buffered in shared memory).  The v1 warp
// kernel held a whole 4096-wide row per warp in 237 registers at 8 warps/SM
// and issued the delta loads one vector at a time (0.52 of HBM).
template <int NT>
__device__ __forceinline__ float row_sum_db(float v, float (&red)[2][NT / 32], int it) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if ((threadIdx.x & 31) == 0) red[it & 1][threadIdx.x >> 5] = v;
    __syncthreads();
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) s += red[it & 1][i];
    return s;
}

template <int NT, int VPT>
__global__ void __launch_bounds__(NT) rmsnorm_fwd_v2_kernel(const __nv_bfloat16* __restrict__ x,
                                                            const __nv_bfloat16* __restrict__ delta,
                                                            __nv_bfloat16* __restrict__ x_out,
                                                            const float* __restrict__ w, float eps,
                                                            __nv_bfloat16* __restrict__ y, float* __restrict__ rstd,
                                                            uint32_t* amax, int T, int d) {
    __shared__ float red[2][NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    const int tid = threadIdx.x;
    float wv[VPT][8];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int c = (i * NT + tid) * 8;
        const float4 a = __ldg(reinterpret_cast<const float4*>(w + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(w + c + 4));
        wv[i][0] = a.x; wv[i][1] = a.y; wv[i][2] = a.z; wv[i][3] = a.w;
        wv[i][4] = b.x; wv[i][5] = b.y; wv[i][6] = b.z; wv[i][7] = b.w;
    }
    uint32_t m = 0;
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
        const int64_t row = (int64_t)t * d;
        uint4 v[VPT], dd[VPT];
#pragma unroll
        for (int i = 0; i < VPT; ++i) v[i] = *reinterpret_cast<const uint4*>(x + row + (i * NT + tid) * 8);
        if (delta) {
#pragma unroll
            for (int i = 0; i < VPT; ++i) dd[i] = *reinterpret_cast<const uint4*>(delta + row + (i * NT + tid) * 8);
        }
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            float a[8];
            unpack_bf16x8(v[i], a);
            if (delta) {
                float b[8];
                unpack_bf16x8(dd[i], b);
#pragma unroll
                for (int j = 0; j < 8; ++j) a[j] += b[j];
                v[i] = bf16x8_pack(a);
                *reinterpret_cast<uint4*>(x_out + row + (i * NT + tid) * 8) = v[i];
                unpack_bf16x8(v[i], a);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) ss = fmaf(a[j], a[j], ss);
        }
        ss = row_sum_db<NT>(ss, red, it);
        const float r = rsqrtf(ss / (float)d + eps);
        if (tid == 0) rstd[t] = r;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            float a[8];
            unpack_bf16x8(v[i], a);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] * r * wv[i][j];
            const uint4 ob = bf16x8_pack(a);
            *reinterpret_cast<uint4*>(y + row + (i * NT + tid) * 8) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    block_amax_commit(m, red_u, amax);
}

template <int NT, int VPT>
__global__ void __launch_bounds__(NT) rmsnorm_bwd_v2_kernel(const __nv_bfloat16* __restrict__ dy,
                                                            const __nv_bfloat16* __restrict__ x,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ rstd,
                                                            const __nv_bfloat16* __restrict__ d_res,
                                                            __nv_bfloat16* __restrict__ dx,
                                                            float* __restrict__ dw_part, uint32_t* amax, int T,
                                                            int d) {
    __shared__ float red[2][NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    const int tid = threadIdx.x;
    float dwp[VPT][8];
#pragma unroll
    for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) dwp[i][j] = 0.f;
    uint32_t m = 0;
    const float inv_d = 1.0f / (float)d;
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++it) {
        const int64_t row = (int64_t)t * d;
        uint4 yv[VPT], xv[VPT], rv[VPT];
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            yv[i] = *reinterpret_cast<const uint4*>(dy + row + (i * NT + tid) * 8);
            xv[i] = *reinterpret_cast<const uint4*>(x + row + (i * NT + tid) * 8);
        }
        if (d_res) {
#pragma unroll
            for (int i = 0; i < VPT; ++i) rv[i] = *reinterpret_cast<const uint4*>(d_res + row + (i * NT + tid) * 8);
        }
        const float r = rstd[t];
        float dot = 0.f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int c = (i * NT + tid) * 8;
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float dv[8], xh[8];
            unpack_bf16x8(yv[i], dv);
            unpack_bf16x8(xv[i], xh);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                xh[j] *= r;
                dot = fmaf(dv[j] * wv[j], xh[j], dot);
                dwp[i][j] = fmaf(dv[j], xh[j], dwp[i][j]);
            }
        }
        dot = row_sum_db<NT>(dot, red, it) * inv_d;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int c = (i * NT + tid) * 8;
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float dv[8], xh[8], o[8];
            unpack_bf16x8(yv[i], dv);
            unpack_bf16x8(xv[i], xh);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                xh[j] *= r;
                o[j] = r * (dv[j] * wv[j] - xh[j] * dot);
            }
            if (d_res) {
                float rr[8];
                unpack_bf16x8(rv[i], rr);
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] += rr[j];
            }
            const uint4 ob = bf16x8_pack(o);
            *reinterpret_cast<uint4*>(dx + row + c) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    if (dw_part) {   // this CTA's column sums; reduced in a fixed order by rmsnorm_dw_reduce_kernel
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            float* dst = dw_part + (int64_t)blockIdx.x * d + (i * NT + tid) * 8;
            reinterpret_cast<float4*>(dst)[0] = make_float4(dwp[i][0], dwp[i][1], dwp[i][2], dwp[i][3]);
            reinterpret_cast<float4*>(dst)[1] = make_float4(dwp[i][4], dwp[i][5], dwp[i][6], dwp[i][7]);
        }
    }
    block_amax_commit(m, red_u, amax);
}

// ---- v3 (d = NT*VPT*8): the v2 dataflow fed by a TMA bulk-copy ring.  Thread 0
// streams whole input rows (cp.async.bulk, 8 KB each at d = 4096) into STAGES
// shared-memory slots ahead of the compute, so every CTA keeps STAGES rows in
// flight regardless of register pressure (v2 had one row in flight per CTA and
// stalled between its load and store phases: 3.3-3.6 TB/s on the bwd).  The
// slot is refilled right after the row-sum barrier (every thread has its
// values in registers by then).
template <int NIN, int STAGES>
struct RowRing {
    uint64_t* full;
    uint8_t* slots;
    int rowb;
    __device__ __forceinline__ uint8_t* slot(int s) const { return slots + (size_t)s * NIN * rowb; }
    __device__ __forceinline__ void issue(int s, const __nv_bfloat16* const (&src)[NIN], int64_t off) const {
        mbar_arrive_expect_tx(&full[s], (uint32_t)(NIN * rowb));
#pragma unroll
        for (int k = 0; k < NIN; ++k)
            if (src[k]) bulk_load(slot(s) + k * rowb, src[k] + off, (uint32_t)rowb, &full[s]);
    }
};

template <int NT, int VPT, int STAGES>
__global__ void __launch_bounds__(NT) rmsnorm_fwd_v3_kernel(const __nv_bfloat16* __restrict__ x,
                                                            const __nv_bfloat16* __restrict__ delta,
                                                            __nv_bfloat16* __restrict__ x_out,
                                                            const float* __restrict__ w, float eps,
                                                            __nv_bfloat16* __restrict__ y, float* __restrict__ rstd,
                                                            uint32_t* amax, int T, int d) {
    extern __shared__ __align__(128) uint8_t rs_smem[];
    constexpr int ROWB = NT * VPT * 16;
    __shared__ float red[2][NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int tid = threadIdx.x, G = gridDim.x;
    const int n = T > (int)blockIdx.x ? (T - (int)blockIdx.x + G - 1) / G : 0;
    RowRing<2, STAGES> ring{full, rs_smem, ROWB};
    // delta absent: the second input slot is simply not loaded (its bytes not expected)
    const __nv_bfloat16* const src[2] = {x, delta};
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int nin_bytes = delta ? 2 * ROWB : ROWB;
    auto issue = [&](int j) {
        const int s = j % STAGES;
        mbar_arrive_expect_tx(&full[s], (uint32_t)nin_bytes);
        const int64_t off = (int64_t)((int)blockIdx.x + j * G) * d;
        bulk_load(ring.slot(s), src[0] + off, ROWB, &full[s]);
        if (delta) bulk_load(ring.slot(s) + ROWB, src[1] + off, ROWB, &full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < min(n, STAGES); ++j) issue(j);
    float wv[VPT][8];
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
        const int c = (i * NT + tid) * 8;
        const float4 a = __ldg(reinterpret_cast<const float4*>(w + c));
        const float4 b = __ldg(reinterpret_cast<const float4*>(w + c + 4));
        wv[i][0] = a.x; wv[i][1] = a.y; wv[i][2] = a.z; wv[i][3] = a.w;
        wv[i][4] = b.x; wv[i][5] = b.y; wv[i][6] = b.z; wv[i][7] = b.w;
    }
    uint32_t m = 0, par = 0;
    for (int j = 0; j < n; ++j) {
        const int s = j % STAGES, t = (int)blockIdx.x + j * G;
        const int64_t row = (int64_t)t * d;
        mbar_wait(&full[s], (par >> s) & 1u);
        par ^= 1u << s;
        const uint32_t base = smem_u32(ring.slot(s));
        uint4 v[VPT];
        float ss = 0.f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            v[i] = lds128(base + (i * NT + tid) * 16);
            float a[8];
            unpack_bf16x8(v[i], a);
            if (delta) {
                float b[8];
                unpack_bf16x8(lds128(base + ROWB + (i * NT + tid) * 16), b);
#pragma unroll
                for (int k = 0; k < 8; ++k) a[k] += b[k];
                v[i] = bf16x8_pack(a);
                *reinterpret_cast<uint4*>(x_out + row + (i * NT + tid) * 8) = v[i];
                unpack_bf16x8(v[i], a);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) ss = fmaf(a[k], a[k], ss);
        }
        ss = row_sum_db<NT>(ss, red, j);             // every thread has read slot s
        if (tid == 0 && j + STAGES < n) issue(j + STAGES);
        const float r = rsqrtf(ss / (float)d + eps);
        if (tid == 0) rstd[t] = r;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            float a[8];
            unpack_bf16x8(v[i], a);
#pragma unroll
            for (int k = 0; k < 8; ++k) a[k] = a[k] * r * wv[i][k];
            const uint4 ob = bf16x8_pack(a);
            *reinterpret_cast<uint4*>(y + row + (i * NT + tid) * 8) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    block_amax_commit(m, red_u, amax);
}

template <int NT, int VPT, int STAGES>
__global__ void __launch_bounds__(NT) rmsnorm_bwd_v3_kernel(const __nv_bfloat16* __restrict__ dy,
                                                            const __nv_bfloat16* __restrict__ x,
                                                            const float* __restrict__ w,
                                                            const float* __restrict__ rstd,
                                                            const __nv_bfloat16* __restrict__ d_res,
                                                            __nv_bfloat16* __restrict__ dx,
                                                            float* __restrict__ dw_part, uint32_t* amax, int T,
                                                            int d) {
    extern __shared__ __align__(128) uint8_t rs_smem[];
    constexpr int ROWB = NT * VPT * 16;
    __shared__ float red[2][NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int tid = threadIdx.x, G = gridDim.x;
    const int n = T > (int)blockIdx.x ? (T - (int)blockIdx.x + G - 1) / G : 0;
    RowRing<3, STAGES> ring{full, rs_smem, ROWB};
    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    const int nbytes = d_res ? 3 * ROWB : 2 * ROWB;
    auto issue = [&](int j) {
        const int s = j % STAGES;
        mbar_arrive_expect_tx(&full[s], (uint32_t)nbytes);
        const int64_t off = (int64_t)((int)blockIdx.x + j * G) * d;
        bulk_load(ring.slot(s), dy + off, ROWB, &full[s]);
        bulk_load(ring.slot(s) + ROWB, x + off, ROWB, &full[s]);
        if (d_res) bulk_load(ring.slot(s) + 2 * ROWB, d_res + off, ROWB, &full[s]);
    };
    if (tid == 0)
        for (int j = 0; j < min(n, STAGES); ++j) issue(j);
    float dwp[VPT][8];
#pragma unroll
    for (int i = 0; i < VPT; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) dwp[i][k] = 0.f;
    uint32_t m = 0, par = 0;
    const float inv_d = 1.0f / (float)d;
    for (int j = 0; j < n; ++j) {
        const int s = j % STAGES, t = (int)blockIdx.x + j * G;
        const int64_t row = (int64_t)t * d;
        const float r = rstd[t];
        mbar_wait(&full[s], (par >> s) & 1u);
        par ^= 1u << s;
        const uint32_t base = smem_u32(ring.slot(s));
        uint4 yv[VPT], xv[VPT], rv[VPT];
        float dot = 0.f;
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int c = (i * NT + tid) * 8;
            yv[i] = lds128(base + (i * NT + tid) * 16);
            xv[i] = lds128(base + ROWB + (i * NT + tid) * 16);
            if (d_res) rv[i] = lds128(base + 2 * ROWB + (i * NT + tid) * 16);
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float dv[8], xh[8];
            unpack_bf16x8(yv[i], dv);
            unpack_bf16x8(xv[i], xh);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                xh[k] *= r;
                dot = fmaf(dv[k] * wv[k], xh[k], dot);
                dwp[i][k] = fmaf(dv[k], xh[k], dwp[i][k]);
            }
        }
        dot = row_sum_db<NT>(dot, red, j) * inv_d;      // every thread has read slot s
        if (tid == 0 && j + STAGES < n) issue(j + STAGES);
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            const int c = (i * NT + tid) * 8;
            const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + c));
            const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + c + 4));
            const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
            float dv[8], xh[8], o[8];
            unpack_bf16x8(yv[i], dv);
            unpack_bf16x8(xv[i], xh);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                xh[k] *= r;
                o[k] = r * (dv[k] * wv[k] - xh[k] * dot);
            }
            if (d_res) {
                float rr[8];
                unpack_bf16x8(rv[i], rr);
#pragma unroll
                for (int k = 0; k < 8; ++k) o[k] += rr[k];
            }
            const uint4 ob = bf16x8_pack(o);
            *reinterpret_cast<uint4*>(dx + row + c) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    if (dw_part) {
#pragma unroll
        for (int i = 0; i < VPT; ++i) {
            float* dst = dw_part + (int64_t)blockIdx.x * d + (i * NT + tid) * 8;
            reinterpret_cast<float4*>(dst)[0] = make_float4(dwp[i][0], dwp[i][1], dwp[i][2], dwp[i][3]);
            reinterpret_cast<float4*>(dst)[1] = make_float4(dwp[i][4], dwp[i][5], dwp[i][6], dwp[i][7]);
        }
    }
    block_amax_commit(m, red_u, amax);
}

// backward: xh = f32(x') * rstd; gw = f32(dy) * w; c = mean(gw * xh)
//   dx = bf16( rstd * (gw - xh * c) + f32(d_res) )   (d_res: gradient arriving
//        through the residual stream; null = 0)
//   dw += sum_t f32(dy) * xh   (per-CTA column sums, then a fixed-order
//        reduction: deterministic, so replays and DP ranks agree bit for bit)
//   amax = max |dx|
template <int NT>
__global__ void __launch_bounds__(NT, (1024 / NT > 0 ? 1024 / NT : 1)) rmsnorm_bwd_kernel(const __nv_bfloat16* __restrict__ dy,
                                                         const __nv_bfloat16* __restrict__ x,
                                                         const float* __restrict__ w, const float* __restrict__ rstd,
                                                         const __nv_bfloat16* __restrict__ d_res,
                                                         __nv_bfloat16* __restrict__ dx, float* __restrict__ dw_part,
                                                         uint32_t* amax, int T, int d) {
    __shared__ float red[NT / 32];
    __shared__ uint32_t red_u[NT / 32];
    const int c = threadIdx.x * 8;
    const bool act = c < d;
    float wv[8], dwp[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (act) {
        const float4 a = *reinterpret_cast<const float4*>(w + c);
        const float4 b = *reinterpret_cast<const float4*>(w + c + 4);
        wv[0] = a.x; wv[1] = a.y; wv[2] = a.z; wv[3] = a.w; wv[4] = b.x; wv[5] = b.y; wv[6] = b.z; wv[7] = b.w;
    }
    uint32_t m = 0;
    const float inv_d = 1.0f / (float)d;
    uint4 ya = make_uint4(0, 0, 0, 0), xa = ya, ra = ya;
    auto load = [&](int t, uint4& yr, uint4& xr, uint4& rr) {
        if (act && t < T) {
            const int64_t off = (int64_t)t * d + c;
            yr = *reinterpret_cast<const uint4*>(dy + off);
            xr = *reinterpret_cast<const uint4*>(x + off);
            if (d_res) rr = *reinterpret_cast<const uint4*>(d_res + off);
        }
    };
    load(blockIdx.x, ya, xa, ra);
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int64_t off = (int64_t)t * d + c;
        uint4 yn = make_uint4(0, 0, 0, 0), xn = yn, rn = yn;
        load(t + gridDim.x, yn, xn, rn);
        const float r = rstd[t];
        float g[8], xh[8];
        float dot = 0.f;
        if (act) {
            float dv[8];
            unpack_bf16x8(ya, dv);
            unpack_bf16x8(xa, xh);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                xh[i] *= r;
                g[i] = dv[i] * wv[i];
                dot = fmaf(g[i], xh[i], dot);
                dwp[i] = fmaf(dv[i], xh[i], dwp[i]);
            }
        }
        dot = block_sum<NT>(dot, red) * inv_d;
        if (act) {
            float o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = r * (g[i] - xh[i] * dot);
            if (d_res) {
                float rv[8];
                unpack_bf16x8(ra, rv);
#pragma unroll
                for (int i = 0; i < 8; ++i) o[i] += rv[i];
            }
            const uint4 ob = bf16x8_pack(o);
            *reinterpret_cast<uint4*>(dx + off) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
        ya = yn;
        xa = xn;
        ra = rn;
    }
    if (act && dw_part) {   // this CTA's column sums; reduced in a fixed order by rmsnorm_dw_reduce_kernel
        float* dst = dw_part + (int64_t)blockIdx.x * d + c;
        reinterpret_cast<float4*>(dst)[0] = make_float4(dwp[0], dwp[1], dwp[2], dwp[3]);
        reinterpret_cast<float4*>(dst)[1] = make_float4(dwp[4], dwp[5], dwp[6], dwp[7]);
    }
    block_amax_commit(m, red_u, amax);
}

// dw[c] += sum_b part[b, c]: thread (cx, ry) of a 64 x 16 block sums rows
// ry, ry+16, ... of column c, then the 16 partial sums are added in ry order
// (a fixed order: deterministic).
__global__ void __launch_bounds__(1024) rmsnorm_dw_reduce_kernel(const float* __restrict__ part, float* __restrict__ dw,
                                                                 int nb, int d) {
    __shared__ float red[16][64];
    const int cx = threadIdx.x & 63, ry = threadIdx.x >> 6;
    const int c = blockIdx.x * 64 + cx;
    float s = 0.f;
    if (c < d)
        for (int b = ry; b < nb; b += 16) s += part[(int64_t)b * d + c];
    red[ry][cx] = s;
    __syncthreads();
    if (ry == 0 && c < d) {
        float t = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) t += red[i][cx];
        dw[c] += t;
    }
}

// ------------------------------------------------------------------ SwiGLU
// gu [T, 2f] = [gate | up];  h = bf16( silu(g) * u ),  amax = max |h|
// grid (column chunks, row groups); each thread one 8-element vector per row
__global__ void __launch_bounds__(256) swiglu_fwd_kernel(const __nv_bfloat16* __restrict__ gu,
                                                         __nv_bfloat16* __restrict__ h, uint32_t* amax, int64_t T,
                                                         int f) {
    __shared__ uint32_t red_u[8];
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    uint32_t m = 0;
    if (c < f) {
        for (int64_t t = blockIdx.y; t < T; t += gridDim.y) {
            float g[8], u[8], o[8];
            bf16x8_load(gu + t * 2 * f + c, g);
            bf16x8_load(gu + t * 2 * f + f + c, u);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = __fdividef(g[k], 1.0f + __expf(-g[k])) * u[k];
            const uint4 ob = bf16x8_pack(o);
            *reinterpret_cast<uint4*>(h + t * f + c) = ob;
            m = max(m, absmax_bits_bf16(ob));
        }
    }
    block_amax_commit(m, red_u, amax);
}

// dh [T, f] -> dgu [T, 2f]:  dg = dh * u * s * (1 + g (1 - s)),  du = dh * g * s,  s = sigmoid(g)
__global__ void __launch_bounds__(256) swiglu_bwd_kernel(const __nv_bfloat16* __restrict__ dh,
                                                         const __nv_bfloat16* __restrict__ gu,
                                                         __nv_bfloat16* __restrict__ dgu, uint32_t* amax, int64_t T,
                                                         int f) {
    __shared__ uint32_t red_u[8];
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    uint32_t m = 0;
    if (c < f) {
        for (int64_t t = blockIdx.y; t < T; t += gridDim.y) {
            float g[8], u[8], d[8], og[8], ou[8];
            bf16x8_load(gu + t * 2 * f + c, g);
            bf16x8_load(gu + t * 2 * f + f + c, u);
            bf16x8_load(dh + t * f + c, d);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float s = __fdividef(1.0f, 1.0f + __expf(-g[k]));
                og[k] = d[k] * u[k] * s * (1.0f + g[k] * (1.0f - s));
                ou[k] = d[k] * g[k] * s;
            }
            const uint4 a = bf16x8_pack(og), b = bf16x8_pack(ou);
            *reinterpret_cast<uint4*>(dgu + t * 2 * f + c) = a;
            *reinterpret_cast<uint4*>(dgu + t * 2 * f + f + c) = b;
            m = max(m, max(absmax_bits_bf16(a), absmax_bits_bf16(b)));
        }
    }
    block_amax_commit(m, red_u, amax);
}

// ------------------------------------------------------------------ RoPE
// qkv [B, S, 3, H, hd] (the qkv projection output) -> q, k, v [B, H, S, hd]
// with q, k rotated by (cos, sin)[s, i] on the pairs (2i, 2i+1):
//   (a, b) -> (a c - b s, a s + b c)
__global__ void __launch_bounds__(256) rope_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       const float* __restrict__ cosv, const float* __restrict__ sinv,
                                                       __nv_bfloat16* __restrict__ q, __nv_bfloat16* __restrict__ k,
                                                       __nv_bfloat16* __restrict__ v, int B, int S, int H, int hd,
                                                       int bshd) {
    // blockIdx.x = token (b, s); (blockIdx.y, thread) cover the H*hd/8 vectors of q, k and v;
    // q, k, v are [B, H, S, hd] contiguous (bshd = 0) or [B, S, H, hd] memory (bshd = 1: what
    // cuDNN SDPA keeps for its output, so the O projection reads it without a transpose copy)
    const int vh = hd / 8;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    if (i >= H * vh) return;
    const int bs = blockIdx.x;
    const int s = bs % S, b = bs / S;
    const int h = i / vh, j = i - h * vh;
    const int64_t src = (int64_t)bs * 3 * H * hd + (int64_t)i * 8;
    const int64_t dst = bshd ? (int64_t)bs * H * hd + (int64_t)i * 8 : (((int64_t)b * H + h) * S + s) * hd + j * 8;
    const float4 c4 = *reinterpret_cast<const float4*>(cosv + (int64_t)s * (hd / 2) + j * 4);
    const float4 s4 = *reinterpret_cast<const float4*>(sinv + (int64_t)s * (hd / 2) + j * 4);
    const float cs[4] = {c4.x, c4.y, c4.z, c4.w}, sn[4] = {s4.x, s4.y, s4.z, s4.w};
    float qa[8], ka[8], qo[8], ko[8];
    bf16x8_load(qkv + src, qa);
    bf16x8_load(qkv + src + (int64_t)H * hd, ka);
    const uint4 vv = *reinterpret_cast<const uint4*>(qkv + src + 2 * (int64_t)H * hd);
#pragma unroll
    for (int p = 0; p < 4; ++p) {
        qo[2 * p] = qa[2 * p] * cs[p] - qa[2 * p + 1] * sn[p];
        qo[2 * p + 1] = qa[2 * p] * sn[p] + qa[2 * p + 1] * cs[p];
        ko[2 * p] = ka[2 * p] * cs[p] - ka[2 * p + 1] * sn[p];
        ko[2 * p + 1] = ka[2 * p] * sn[p] + ka[2 * p + 1] * cs[p];
    }
    *reinterpret_cast<uint4*>(q + dst) = bf16x8_pack(qo);
    *reinterpret_cast<uint4*>(k + dst) = bf16x8_pack(ko);
    *reinterpret_cast<uint4*>(v + dst) = vv;
}

// dq, dk, dv [B, H, S, hd] -> dqkv [B, S, 3, H, hd] (inverse rotation), amax = max |dqkv|
__global__ void __launch_bounds__(256) rope_bwd_kernel(const __nv_bfloat16* __restrict__ dq,
                                                       const __nv_bfloat16* __restrict__ dk,
                                                       const __nv_bfloat16* __restrict__ dv,
                                                       const float* __restrict__ cosv, const float* __restrict__ sinv,
                                                       __nv_bfloat16* __restrict__ dqkv, uint32_t* amax, int B, int S,
                                                       int H, int hd, int bshd) {
    __shared__ uint32_t red_u[8];
    const int vh = hd / 8;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    uint32_t m = 0;
    if (i < H * vh) {
        const int bs = blockIdx.x;
        const int s = bs % S, b = bs / S;
        const int h = i / vh, j = i - h * vh;
        const int64_t dst = (int64_t)bs * 3 * H * hd + (int64_t)i * 8;
        const int64_t src = bshd ? (int64_t)bs * H * hd + (int64_t)i * 8 : (((int64_t)b * H + h) * S + s) * hd + j * 8;
        const float4 c4 = *reinterpret_cast<const float4*>(cosv + (int64_t)s * (hd / 2) + j * 4);
        const float4 s4 = *reinterpret_cast<const float4*>(sinv + (int64_t)s * (hd / 2) + j * 4);
        const float cs[4] = {c4.x, c4.y, c4.z, c4.w}, sn[4] = {s4.x, s4.y, s4.z, s4.w};
        float qa[8], ka[8], qo[8], ko[8];
        bf16x8_load(dq + src, qa);
        bf16x8_load(dk + src, ka);
        const uint4 vv = *reinterpret_cast<const uint4*>(dv + src);
#pragma unroll
        for (int p = 0; p < 4; ++p) {
            qo[2 * p] = qa[2 * p] * cs[p] + qa[2 * p + 1] * sn[p];
            qo[2 * p + 1] = -qa[2 * p] * sn[p] + qa[2 * p + 1] * cs[p];
            ko[2 * p] = ka[2 * p] * cs[p] + ka[2 * p + 1] * sn[p];
            ko[2 * p + 1] = -ka[2 * p] * sn[p] + ka[2 * p + 1] * cs[p];
        }
        const uint4 a = bf16x8_pack(qo), bb = bf16x8_pack(ko);
        *reinterpret_cast<uint4*>(dqkv + dst) = a;
        *reinterpret_cast<uint4*>(dqkv + dst + (int64_t)H * hd) = bb;
        *reinterpret_cast<uint4*>(dqkv + dst + 2 * (int64_t)H * hd) = vv;
        m = max(absmax_bits_bf16(a), max(absmax_bits_bf16(bb), absmax_bits_bf16(vv)));
    }
    block_amax_commit(m, red_u, amax);
}

// ------------------------------------------------------------------ small glue producers (LayerStack)
// mode 0: sum3   out [T, d] = a + b + c from x [T, 3d] (column blocks), amax(out)
// mode 1: bcast3 out [T, 3d] = [x, x, x] from x [T, d],               amax(x)
// mode 2: add    out [T, d] = x + y,                                  amax(out)
// mode 3: mse'   out [T, d] = x * f32(*scale * alpha),                amax(out)   (dL/dy of mean(y^2): *scale = g, alpha = 2/n)
// Each thread owns 8 columns and walks rows with stride gridDim.y, GLUE_R rows
// per iteration: all 16-byte loads of the R rows are issued before any math
// (memory-level parallelism; one row per iteration left the 2-input add at
// 49 % of HBM peak).
constexpr int GLUE_R = 4;
template <int MODE>
__global__ void __launch_bounds__(256) glue_kernel(const __nv_bfloat16* __restrict__ x,
                                                   const __nv_bfloat16* __restrict__ y, const float* __restrict__ scale,
                                                   float alpha, __nv_bfloat16* __restrict__ out, uint32_t* amax,
                                                   int64_t T, int d) {
    constexpr int NIN = MODE == 0 ? 3 : (MODE == 2 || MODE == 3) ? 2 : 1;   // mode 3: y optional (offset)
    __shared__ uint32_t red_u[8];
    const int c = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
    uint32_t m = 0;
    const float sc = MODE == 3 ? *scale * alpha : 0.f;
    const int64_t in_ld = MODE == 0 ? 3 * (int64_t)d : d;
    const int64_t out_ld = MODE == 1 ? 3 * (int64_t)d : d;
    if (c < d) {
        for (int64_t t0 = blockIdx.y; t0 < T; t0 += (int64_t)gridDim.y * GLUE_R) {
            uint4 in[GLUE_R][NIN];
#pragma unroll
            for (int r = 0; r < GLUE_R; ++r) {
                const int64_t t = t0 + (int64_t)r * gridDim.y;
                if (t < T) {
                    const __nv_bfloat16* px = x + t * in_ld + c;
#pragma unroll
                    for (int j = 0; j < NIN; ++j) {
                        if (MODE == 3 && j == 1) {
                            if (y) in[r][1] = *reinterpret_cast<const uint4*>(y + t * d + c);
                        } else {
                            in[r][j] = *reinterpret_cast<const uint4*>((MODE == 2 && j == 1) ? y + t * d + c : px + j * d);
                        }
                    }
                }
            }
#pragma unroll
            for (int r = 0; r < GLUE_R; ++r) {
                const int64_t t = t0 + (int64_t)r * gridDim.y;
                if (t >= T) break;
                float a[8];
                unpack_bf16x8(in[r][0], a);
                if (MODE == 0 || MODE == 2) {
#pragma unroll
                    for (int j = 1; j < NIN; ++j) {
                        float b[8];
                        unpack_bf16x8(in[r][j], b);
#pragma unroll
                        for (int k = 0; k < 8; ++k) a[k] += b[k];
                    }
                } else if (MODE == 3) {
                    if (y) {                                   // out = (x + y) * scale
                        float b[8];
                        unpack_bf16x8(in[r][1], b);
#pragma unroll
                        for (int k = 0; k < 8; ++k) a[k] += b[k];
                    }
#pragma unroll
                    for (int k = 0; k < 8; ++k) a[k] *= sc;
                }
                const uint4 o = MODE == 1 ? in[r][0] : bf16x8_pack(a);
                __nv_bfloat16* po = out + t * out_ld + c;
                *reinterpret_cast<uint4*>(po) = o;
                if (MODE == 1) {
                    *reinterpret_cast<uint4*>(po + d) = o;
                    *reinterpret_cast<uint4*>(po + 2 * d) = o;
                }
                m = max(m, absmax_bits_bf16(o));
            }
        }
    }
    block_amax_commit(m, red_u, amax);
}

// sum of squares of a bf16 tensor in f32, deterministic: per-CTA partials in a
// fixed-size buffer, then one CTA reduces them in a fixed order (no atomics:
// the loss is bit-reproducible across runs and CUDA-graph replays)
constexpr int SUMSQ_PARTS = 1024;
__global__ void __launch_bounds__(256) sumsq_kernel(const __nv_bfloat16* __restrict__ x,
                                                    const __nv_bfloat16* __restrict__ y, int64_t nvec,
                                                    float* __restrict__ parts) {
    __shared__ float red[8];
    float ssum = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (int64_t)gridDim.x * blockDim.x) {
        float v[8];
        bf16x8_load(x + i * 8, v);
        if (y) {                                                // sum (x + y)^2, y a fixed offset
            float b[8];
            bf16x8_load(y + i * 8, b);
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] += b[k];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) ssum = fmaf(v[k], v[k], ssum);
    }
    ssum = block_sum<256>(ssum, red);
    if (threadIdx.x == 0) parts[blockIdx.x] = ssum;
}

__global__ void __launch_bounds__(SUMSQ_PARTS) sumsq_final_kernel(const float* __restrict__ parts, int n,
                                                                  float scale, float* __restrict__ acc) {
    __shared__ float red[SUMSQ_PARTS / 32];
    float v = threadIdx.x < n ? parts[threadIdx.x] : 0.f;
    v = block_sum<SUMSQ_PARTS>(v, red);
    if (threadIdx.x == 0) *acc = v * scale;
}

// ------------------------------------------------------------------ cross entropy (LM head)
// forward: one CTA per row of bf16 logits [T, V]: online max / sum-exp in f32
// (one read of the row), lse[t] = max + log(sum), loss[t] = lse[t] - x[t, y_t]
__global__ void __launch_bounds__(256) xent_fwd_kernel(const __nv_bfloat16* __restrict__ logits,
                                                       const int64_t* __restrict__ targets, float* __restrict__ lse,
                                                       float* __restrict__ loss, int V) {
    __shared__ float red_m[8], red_s[8];
    const int64_t t = blockIdx.x;
    const __nv_bfloat16* row = logits + t * V;
    float m = -INFINITY, sum = 0.f;
    const int nv = V / 8;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        float v[8];
        bf16x8_load(row + i * 8, v);
        float vm = v[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) vm = fmaxf(vm, v[j]);
        const float nm = fmaxf(m, vm);
        sum *= __expf(m - nm);
#pragma unroll
        for (int j = 0; j < 8; ++j) sum += __expf(v[j] - nm);
        m = nm;
    }
    // merge (m, sum) pairs: warp, then CTA
    // (threads without elements carry (-inf, 0): their terms are skipped, exp(-inf - -inf) would be NaN)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float om = __shfl_xor_sync(0xFFFFFFFFu, m, o), os = __shfl_xor_sync(0xFFFFFFFFu, sum, o);
        const float nm = fmaxf(m, om);
        sum = (m == -INFINITY ? 0.f : sum * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
        m = nm;
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red_m[warp] = m;
        red_s[warp] = sum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float M = red_m[0], S = red_s[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            if (red_m[w] == -INFINITY) continue;
            const float nm = fmaxf(M, red_m[w]);
            S = (M == -INFINITY ? 0.f : S * __expf(M - nm)) + red_s[w] * __expf(red_m[w] - nm);
            M = nm;
        }
        const float l = M + __logf(S);
        lse[t] = l;
        loss[t] = l - __bfloat162float(row[targets[t]]);
    }
}

// backward: dlogits[t, v] = (exp(x - lse[t]) - [v == y_t]) * (*scale)   (scale = dL/dloss / T)
__global__ void __launch_bounds__(256) xent_bwd_kernel(const __nv_bfloat16* __restrict__ logits,
                                                       const int64_t* __restrict__ targets,
                                                       const float* __restrict__ lse, const float* __restrict__ scale,
                                                       __nv_bfloat16* __restrict__ dlogits, int V) {
    const int64_t t = blockIdx.x;
    const float l = lse[t], sc = *scale;
    const int64_t y = targets[t];
    const __nv_bfloat16* row = logits + t * V;
    __nv_bfloat16* out = dlogits + t * V;
    for (int i = threadIdx.x; i < V / 8; i += blockDim.x) {
        float v[8];
        bf16x8_load(row + i * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = (__expf(v[j] - l) - ((int64_t)(i * 8 + j) == y ? 1.f : 0.f)) * sc;
        *reinterpret_cast<uint4*>(out + i * 8) = bf16x8_pack(v);
    }
}

// ------------------------------------------------------------------ launchers
template <typename K>
static int resident(K kern, int threads) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0) != cudaSuccess || occ < 1) occ = 1;
    return occ;
}

// MOSS_RMS_V2 (A/B testing, d = 4096): 4 (default) the TMA-ring v3 kernels with 256 threads x 2
// vectors per row, 3 = v3 with 128 x 4, 1 = v2 128 x 4, 2 = v2 256 x 2, 0 = the v1 kernels
static int rms_v2_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_RMS_V2");
        v = e ? (e[0] - '0') : 4;
        if (v < 0 || v > 4) v = 4;
    }
    return v;
}
constexpr int RMS3_FWD_STAGES = 4, RMS3_BWD_STAGES = 3;
constexpr int RMS3_FWD_SMEM = RMS3_FWD_STAGES * 2 * 4096 * 2;    // x + delta rows, bf16
constexpr int RMS3_BWD_SMEM = RMS3_BWD_STAGES * 3 * 4096 * 2;    // dy + x + d_res rows

template <int NT>
static int rms3_bwd_occ_t() {
    static int occ_dev[kMaxDevices] = {};
    static bool optin[kMaxDevices] = {};
    const int dev = current_device();
    auto kern = rmsnorm_bwd_v3_kernel<NT, 512 / NT, RMS3_BWD_STAGES>;
    if (!smem_optin(kern, RMS3_BWD_SMEM, optin)) return 0;
    if (!occ_dev[dev] &&
        (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_dev[dev], kern, NT, RMS3_BWD_SMEM) != cudaSuccess ||
         occ_dev[dev] < 1))
        occ_dev[dev] = 1;
    return occ_dev[dev];
}
static int rms3_bwd_occ() { return rms_v2_mode() == 4 ? rms3_bwd_occ_t<256>() : rms3_bwd_occ_t<128>(); }

static dim3 swiglu_grid(int64_t T, int64_t f) {
    const int64_t gx = (f / 8 + 255) / 256;
    const int64_t gy = std::min<int64_t>(T, std::max<int64_t>(1, (int64_t)sm_count() * 16 / gx));
    return dim3((unsigned)gx, (unsigned)gy);
}

static int amax_reset(uint32_t* amax, cudaStream_t st) {
    return (amax && zero_word(amax, st) != cudaSuccess) ? MOSS_ERR_CUDA : MOSS_OK;
}

int launch_rmsnorm_fwd(const void* x, const void* delta, void* x_out, const float* w, float eps, void* y, float* rstd,
                       float* amax, int64_t T, int64_t d, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    if (d == 4096 && rms_v2_mode() != 0) {
        auto go = [&](auto kern, int nt) {
            static int occ = resident(kern, nt);    // one static per kernel instance
            const int grid = (int)std::min<int64_t>(T, (int64_t)sm_count() * occ);
            kern<<<grid, nt, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)delta, (__nv_bfloat16*)x_out,
                                      w, eps, (__nv_bfloat16*)y, rstd, reinterpret_cast<uint32_t*>(amax), (int)T,
                                      (int)d);
        };
        if (rms_v2_mode() >= 3) {
            auto go3 = [&](auto kern, int nt) {
                static bool optin[kMaxDevices] = {};
                static int occ_dev[kMaxDevices] = {};
                const int dev = current_device();
                if (!smem_optin(kern, RMS3_FWD_SMEM, optin)) return false;
                if (!occ_dev[dev] && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_dev[dev], kern, nt,
                                                                                    RMS3_FWD_SMEM) != cudaSuccess ||
                                      occ_dev[dev] < 1))
                    occ_dev[dev] = 1;
                const int grid = (int)std::min<int64_t>(T, (int64_t)sm_count() * occ_dev[dev]);
                kern<<<grid, nt, RMS3_FWD_SMEM, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)delta,
                                                      (__nv_bfloat16*)x_out, w, eps, (__nv_bfloat16*)y, rstd,
                                                      reinterpret_cast<uint32_t*>(amax), (int)T, (int)d);
                return true;
            };
            const bool ok = rms_v2_mode() == 4 ? go3(rmsnorm_fwd_v3_kernel<256, 2, RMS3_FWD_STAGES>, 256)
                                               : go3(rmsnorm_fwd_v3_kernel<128, 4, RMS3_FWD_STAGES>, 128);
            if (!ok) return MOSS_ERR_CUDA;
        } else if (rms_v2_mode() == 2) {
            go(rmsnorm_fwd_v2_kernel<256, 2>, 256);
        } else {
            go(rmsnorm_fwd_v2_kernel<128, 4>, 128);
        }
        return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
    }
    if (d % 256 == 0 && d / 256 <= 16) {
        auto warp_args = [&](auto kern) {
            static int occ = resident(kern, 256);
            const int grid = (int)std::min<int64_t>((T + 7) / 8, (int64_t)sm_count() * occ);
            kern<<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)delta, (__nv_bfloat16*)x_out, w,
                                       eps, (__nv_bfloat16*)y, rstd, reinterpret_cast<uint32_t*>(amax), (int)T, (int)d);
        };
        switch (d / 256) {
            case 1: warp_args(rmsnorm_fwd_warp_kernel<1>); break;
            case 2: warp_args(rmsnorm_fwd_warp_kernel<2>); break;
            case 3: warp_args(rmsnorm_fwd_warp_kernel<3>); break;
            case 4: warp_args(rmsnorm_fwd_warp_kernel<4>); break;
            case 8: warp_args(rmsnorm_fwd_warp_kernel<8>); break;
            case 12: warp_args(rmsnorm_fwd_warp_kernel<12>); break;
            case 16: warp_args(rmsnorm_fwd_warp_kernel<16>); break;
            default: goto block_path;
        }
        return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
    }
block_path:
    const int nt = (int)((d / 8 + 31) / 32 * 32);
    auto args = [&](auto kern) {
        static int occ = resident(kern, nt);     // one static per template instance
        const int grid = (int)std::min<int64_t>(T, (int64_t)sm_count() * occ);
        kern<<<grid, nt, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)delta,
                                                  (__nv_bfloat16*)x_out, w, eps, (__nv_bfloat16*)y, rstd,
                                                  reinterpret_cast<uint32_t*>(amax), (int)T, (int)d);
    };
    switch (nt) {
        case 32: args(rmsnorm_fwd_kernel<32>); break;
        case 64: args(rmsnorm_fwd_kernel<64>); break;
        case 96: args(rmsnorm_fwd_kernel<96>); break;
        case 128: args(rmsnorm_fwd_kernel<128>); break;
        case 256: args(rmsnorm_fwd_kernel<256>); break;
        case 512: args(rmsnorm_fwd_kernel<512>); break;
        case 1024: args(rmsnorm_fwd_kernel<1024>); break;
        default: return MOSS_ERR_SHAPE;
    }
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

static int rmsnorm_bwd_grid(int64_t T, int64_t d) {
    if (d == 4096 && rms_v2_mode() != 0) {
        static int occ1 = resident(rmsnorm_bwd_v2_kernel<128, 4>, 128);
        static int occ2 = resident(rmsnorm_bwd_v2_kernel<256, 2>, 256);
        const int occ = rms_v2_mode() >= 3 ? std::max(1, rms3_bwd_occ()) : rms_v2_mode() == 2 ? occ2 : occ1;
        return (int)std::min<int64_t>(T, (int64_t)sm_count() * occ);
    }
    const int nt = (int)((d / 8 + 31) / 32 * 32);
    return (int)std::min<int64_t>(T, (int64_t)sm_count() * std::max(1, 1024 / nt));
}

int64_t rmsnorm_bwd_workspace(int64_t T, int64_t d) { return (int64_t)rmsnorm_bwd_grid(T, d) * d * 4; }

int launch_rmsnorm_bwd(const void* dy, const void* x, const float* w, const float* rstd, const void* d_res, void* dx,
                       float* dw, float* amax, float* ws, int64_t T, int64_t d, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    const int nt = (int)((d / 8 + 31) / 32 * 32);
    const int grid = rmsnorm_bwd_grid(T, d);
    if (d == 4096 && rms_v2_mode() != 0) {
        auto go = [&](auto kern, int ntv) {
            kern<<<grid, ntv, 0, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, w, rstd,
                                       (const __nv_bfloat16*)d_res, (__nv_bfloat16*)dx, dw ? ws : nullptr,
                                       reinterpret_cast<uint32_t*>(amax), (int)T, (int)d);
        };
        if (rms_v2_mode() >= 3) {
            if (!rms3_bwd_occ()) return MOSS_ERR_CUDA;
            auto go3 = [&](auto kern, int ntv) {
                kern<<<grid, ntv, RMS3_BWD_SMEM, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, w, rstd,
                                                       (const __nv_bfloat16*)d_res, (__nv_bfloat16*)dx,
                                                       dw ? ws : nullptr, reinterpret_cast<uint32_t*>(amax), (int)T,
                                                       (int)d);
            };
            if (rms_v2_mode() == 4) go3(rmsnorm_bwd_v3_kernel<256, 2, RMS3_BWD_STAGES>, 256);
            else go3(rmsnorm_bwd_v3_kernel<128, 4, RMS3_BWD_STAGES>, 128);
        } else if (rms_v2_mode() == 2) {
            go(rmsnorm_bwd_v2_kernel<256, 2>, 256);
        } else {
            go(rmsnorm_bwd_v2_kernel<128, 4>, 128);
        }
        if (dw) rmsnorm_dw_reduce_kernel<<<(unsigned)((d + 63) / 64), 1024, 0, st>>>(ws, dw, grid, (int)d);
        return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
    }
    auto args = [&](auto kern) {
        kern<<<grid, nt, 0, st>>>((const __nv_bfloat16*)dy, (const __nv_bfloat16*)x, w, rstd,
                                  (const __nv_bfloat16*)d_res, (__nv_bfloat16*)dx, dw ? ws : nullptr,
                                  reinterpret_cast<uint32_t*>(amax), (int)T, (int)d);
    };
    switch (nt) {
        case 32: args(rmsnorm_bwd_kernel<32>); break;
        case 64: args(rmsnorm_bwd_kernel<64>); break;
        case 96: args(rmsnorm_bwd_kernel<96>); break;
        case 128: args(rmsnorm_bwd_kernel<128>); break;
        case 256: args(rmsnorm_bwd_kernel<256>); break;
        case 512: args(rmsnorm_bwd_kernel<512>); break;
        case 1024: args(rmsnorm_bwd_kernel<1024>); break;
        default: return MOSS_ERR_SHAPE;
    }
    if (dw) rmsnorm_dw_reduce_kernel<<<(unsigned)((d + 63) / 64), 1024, 0, st>>>(ws, dw, grid, (int)d);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_swiglu_fwd(const void* gu, void* h, float* amax, int64_t T, int64_t f, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    swiglu_fwd_kernel<<<swiglu_grid(T, f), 256, 0, st>>>(
        (const __nv_bfloat16*)gu, (__nv_bfloat16*)h, reinterpret_cast<uint32_t*>(amax), T, (int)f);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_swiglu_bwd(const void* dh, const void* gu, void* dgu, float* amax, int64_t T, int64_t f, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    swiglu_bwd_kernel<<<swiglu_grid(T, f), 256, 0, st>>>(
        (const __nv_bfloat16*)dh, (const __nv_bfloat16*)gu, (__nv_bfloat16*)dgu, reinterpret_cast<uint32_t*>(amax), T,
        (int)f);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_rope_fwd(const void* qkv, const float* cosv, const float* sinv, void* q, void* k, void* v, int64_t B,
                    int64_t S, int64_t H, int64_t hd, int bshd, cudaStream_t st) {
    rope_fwd_kernel<<<dim3((unsigned)(B * S), (unsigned)((H * (hd / 8) + 255) / 256)), 256, 0, st>>>(
        (const __nv_bfloat16*)qkv, cosv, sinv, (__nv_bfloat16*)q, (__nv_bfloat16*)k, (__nv_bfloat16*)v, (int)B, (int)S,
        (int)H, (int)hd, bshd);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_rope_bwd(const void* dq, const void* dk, const void* dv, const float* cosv, const float* sinv, void* dqkv,
                    float* amax, int64_t B, int64_t S, int64_t H, int64_t hd, int bshd, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    rope_bwd_kernel<<<dim3((unsigned)(B * S), (unsigned)((H * (hd / 8) + 255) / 256)), 256, 0, st>>>(
        (const __nv_bfloat16*)dq, (const __nv_bfloat16*)dk, (const __nv_bfloat16*)dv, cosv, sinv,
        (__nv_bfloat16*)dqkv, reinterpret_cast<uint32_t*>(amax), (int)B, (int)S, (int)H, (int)hd, bshd);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_glue(int mode, const void* x, const void* y, const float* scale, float alpha, void* out, float* amax,
                int64_t T, int64_t d, cudaStream_t st) {
    if (amax_reset(reinterpret_cast<uint32_t*>(amax), st)) return MOSS_ERR_CUDA;
    const int64_t gx = (d / 8 + 255) / 256;
    auto kern = mode == 0 ? glue_kernel<0> : mode == 1 ? glue_kernel<1> : mode == 2 ? glue_kernel<2> : glue_kernel<3>;
    static int occ[4] = {resident(glue_kernel<0>, 256), resident(glue_kernel<1>, 256), resident(glue_kernel<2>, 256),
                         resident(glue_kernel<3>, 256)};
    const int64_t gy = std::min<int64_t>((T + GLUE_R - 1) / GLUE_R,
                                         std::max<int64_t>(1, (int64_t)sm_count() * occ[mode] / gx));
    kern<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)y, scale,
                                                           alpha, (__nv_bfloat16*)out, reinterpret_cast<uint32_t*>(amax), T,
                                                           (int)d);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_sumsq(const void* x, const void* y, int64_t n, float scale, float* acc, float* parts, cudaStream_t st) {
    const int64_t nvec = n / 8;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nvec + 255) / 256, SUMSQ_PARTS));
    sumsq_kernel<<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, (const __nv_bfloat16*)y, nvec, parts);
    sumsq_final_kernel<<<1, SUMSQ_PARTS, 0, st>>>(parts, grid, scale, acc);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_xent_fwd(const void* logits, const int64_t* targets, float* lse, float* loss, int64_t T, int64_t V,
                    cudaStream_t st) {
    xent_fwd_kernel<<<(unsigned)T, 256, 0, st>>>((const __nv_bfloat16*)logits, targets, lse, loss, (int)V);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_xent_bwd(const void* logits, const int64_t* targets, const float* lse, const float* scale, void* dlogits,
                    int64_t T, int64_t V, cudaStream_t st) {
    xent_bwd_kernel<<<(unsigned)T, 256, 0, st>>>((const __nv_bfloat16*)logits, targets, lse, scale,
                                                 (__nv_bfloat16*)dlogits, (int)V);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

}  // namespace moss
