// Per-group (COAT-style) FP8 quantizer and main-loop-dequant GEMM — the
// ABLATION COMPARATOR of the paper's Fig. 1 / Table 7 contrast
// (SURVEY.md 8(f) rank 4), not part of the MOSS training path.
//
//   quant_per_group   (reference quantize.py:100-124): one f32 scale per
//                     contiguous group of G = 128 elements along a row,
//                     s = f32(amax/448) (0 -> 1.0), codes = e4m3(x / s)
//   gemm_pergroup     (reference gemm.py:132-157):
//                     C[m, n] = sum_g (A_g B_g^T)[m, n] * sa[m, g] * sb[n, g]
//
// With per-group f32 scales the tensor core cannot apply the scales (the
// block-scaled MMA takes E8M0 per 32, not f32 per 128), so every 128-deep
// partial product has to leave TMEM and be rescaled on the CUDA cores
// ("promotion").  Kernel: one CTA per SM, persistent over 128 x 128 tiles;
// warp 0 TMA producer (A, B tiles + the group's 128 + 128 scales), warp 1
// issues 4 x tcgen05.mma.kind::f8f6f4 (no block scale) per group into one of
// two TMEM partial buffers (ping-pong), warps 4-11 drain each partial
// (tcgen05.ld), release the buffer and accumulate acc += partial * sa * sb
// in registers (FMUL2 + FFMA2), then store the tile.  The MX kernel
// (gemm2.cu) instead accumulates all of K in TMEM and scales once.
#include <algorithm>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

// ------------------------------------------------------------------ quantizer
// one warp per (row, group): 128 elements = 4 per lane
template <typename T>
__global__ void __launch_bounds__(256) quant_per_group_kernel(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                              uint8_t* __restrict__ codes, float* __restrict__ scales,
                                                              uint32_t* flags) {
    const int lane = threadIdx.x & 31;
    const int64_t groups = cols / 128;
    const int64_t total = rows * groups;
    bool bad = false;
    for (int64_t wi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < total;
         wi += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t r = wi / groups, g = wi - r * groups;
        const int64_t off = r * cols + g * 128 + lane * 4;
        float v[4];
        if constexpr (sizeof(T) == 2) {
            const uint2 u = *reinterpret_cast<const uint2*>(x + off);
            v[0] = __uint_as_float(u.x << 16);
            v[1] = __uint_as_float(u.x & 0xFFFF0000u);
            v[2] = __uint_as_float(u.y << 16);
            v[3] = __uint_as_float(u.y & 0xFFFF0000u);
        } else {
            const float4 f = *reinterpret_cast<const float4*>(x + off);
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        }
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            bad |= nonfinite(v[i]);
            m = fmaxf(m, fabsf(v[i]));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        // quantize.py:118-121: s = f32(amax / f32(448)), zero group -> 1.0; codes = encode(block / s)
        const float s = m > 0.f ? __fdiv_rn(m, kE4M3Max) : 1.0f;
        const uint32_t q = e4m3x4(__fdiv_rn(v[0], s), __fdiv_rn(v[1], s), __fdiv_rn(v[2], s), __fdiv_rn(v[3], s));
        *reinterpret_cast<uint32_t*>(codes + off) = q;
        if (lane == 0) scales[r * groups + g] = s;
    }
    if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, MOSS_FLAG_NONFINITE);
}

int launch_quant_per_group(const void* x, int dtype, int64_t rows, int64_t cols, uint8_t* codes, float* scales,
                           uint32_t* flags, cudaStream_t st) {
    const int64_t warps = rows * (cols / 128);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)sm_count() * 8));
    if (dtype == MOSS_BF16)
        quant_per_group_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>((const __nv_bfloat16*)x, rows, cols, codes, scales,
                                                                    flags);
    else
        quant_per_group_kernel<float><<<grid, 256, 0, st>>>((const float*)x, rows, cols, codes, scales, flags);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

// ------------------------------------------------------------------ GEMM
constexpr int PG_BM = 128, PG_BN = 128, PG_BK = 128, PG_STAGES = 4, PG_THREADS = 384, PG_EPI = 8;

struct PgLayout {
    static constexpr int A_BYTES = PG_BM * PG_BK;             // 16 KB
    static constexpr int B_BYTES = PG_BN * PG_BK;             // 16 KB
    static constexpr int S_BYTES = (PG_BM + PG_BN) * 4;        // the group's 128 + 128 f32 scales
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + PG_STAGES * A_BYTES;
    static constexpr int OFF_S = OFF_B + PG_STAGES * B_BYTES;
    static constexpr int OFF_BAR = OFF_S + PG_STAGES * S_BYTES;
    static constexpr int N_BARS = 2 * PG_STAGES + 4;           // full, empty, part_full[2], part_empty[2]
    static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
    static constexpr int SMEM = OFF_TMEM + 16 + 1024;
};

// kind::f8f6f4 instruction descriptor: D f32, A = B = E4M3, K-major, M x N
__host__ __device__ constexpr uint32_t f8_idesc(uint32_t m, uint32_t n) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}

__device__ __forceinline__ void mma_f8(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

// sa_t [G, M], sb_t [G, N]: scales group-major (the wrapper transposes the reference's [M, G])
template <bool OUT_BF16>
__global__ void __launch_bounds__(PG_THREADS, 1)
    gemm_pergroup_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const float* __restrict__ sa_t, const float* __restrict__ sb_t, void* __restrict__ D,
                         int64_t ldd, int M, int N, int K) {
    using L = PgLayout;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_a = smem + L::OFF_A;
    uint8_t* s_b = smem + L::OFF_B;
    float* s_s = reinterpret_cast<float*>(smem + L::OFF_S);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* empty = full + PG_STAGES;
    uint64_t* part_full = empty + PG_STAGES;      // [2]
    uint64_t* part_empty = part_full + 2;         // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tiles = M / PG_BM, n_tiles = N / PG_BN, num_tiles = m_tiles * n_tiles;
    const int kblocks = K / PG_BK;
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < PG_STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1 + PG_EPI);       // the MMA commit + every promotion warp (scales read)
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&part_full[b], 1);
            mbar_init(&part_empty[b], PG_EPI);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mb = tile % m_tiles, nb = tile / m_tiles;
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&full[stage], L::A_BYTES + L::B_BYTES + L::S_BYTES);
                    tma_load_2d(s_a + stage * L::A_BYTES, &tmA, &full[stage], kb * PG_BK, mb * PG_BM);
                    tma_load_2d(s_b + stage * L::B_BYTES, &tmB, &full[stage], kb * PG_BK, nb * PG_BN);
                    float* ss = s_s + stage * (PG_BM + PG_BN);
                    bulk_load(ss, sa_t + (int64_t)kb * M + (int64_t)mb * PG_BM, PG_BM * 4, &full[stage]);
                    bulk_load(ss + PG_BM, sb_t + (int64_t)kb * N + (int64_t)nb * PG_BN, PG_BN * 4, &full[stage]);
                }
                __syncwarp();
                if (++stage == PG_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        int stage = 0, pb = 0;
        uint32_t phase = 0, pphase[2] = {0, 0};
        constexpr uint32_t idesc = f8_idesc(PG_BM, PG_BN);
        const uint64_t adesc0 = umma_desc(smem_u32(s_a), 0, 1024, kLayoutSW128);
        const uint64_t bdesc0 = umma_desc(smem_u32(s_b), 0, 1024, kLayoutSW128);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                mbar_wait(&part_empty[pb], pphase[pb] ^ 1);   // promotion has drained this partial buffer
                pphase[pb] ^= 1;
                tc_fence_after();
                if (elect_one()) {
                    const uint64_t adesc = adesc0 + (uint64_t)((stage * L::A_BYTES) >> 4);
                    const uint64_t bdesc = bdesc0 + (uint64_t)((stage * L::B_BYTES) >> 4);
#pragma unroll
                    for (int k = 0; k < PG_BK / 32; ++k)
                        mma_f8(tmem + pb * PG_BN, adesc + 2 * k, bdesc + 2 * k, idesc, k != 0);   // a fresh partial per group
                    tc_commit(&part_full[pb]);
                    tc_commit(&empty[stage]);
                }
                __syncwarp();
                pb ^= 1;
                if (++stage == PG_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp >= 4) {
        // promotion + epilogue: warp -> TMEM lanes [32 quad, +32), columns [64 half, +64)
        const int ew = warp - 4, quad = warp & 3, half = ew >> 2;
        const int row_in = quad * 32 + lane;
        int stage = 0, pb = 0;
        uint32_t phase = 0, pphase[2] = {0, 0};
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mb = tile % m_tiles, nb = tile / m_tiles;
            float acc[64];
#pragma unroll
            for (int j = 0; j < 64; ++j) acc[j] = 0.f;
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&part_full[pb], pphase[pb]);
                pphase[pb] ^= 1;
                tc_fence_after();
                uint32_t p[64];
                const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + pb * PG_BN + half * 64;
                tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(&p[0]));
                tmem_ld32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&p[32]));
                tmem_ld_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0)
                    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&part_empty[pb]))
                                 : "memory");
                mbar_wait(&full[stage], phase);              // this group's scales are in smem (already complete)
                const float* ss = s_s + stage * (PG_BM + PG_BN);
                const float sa = ss[row_in];
                const float4* sb4 = reinterpret_cast<const float4*>(ss + PG_BM + half * 64);
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    const float4 b = sb4[q];
                    acc[4 * q + 0] = fmaf(__uint_as_float(p[4 * q + 0]), sa * b.x, acc[4 * q + 0]);
                    acc[4 * q + 1] = fmaf(__uint_as_float(p[4 * q + 1]), sa * b.y, acc[4 * q + 1]);
                    acc[4 * q + 2] = fmaf(__uint_as_float(p[4 * q + 2]), sa * b.z, acc[4 * q + 2]);
                    acc[4 * q + 3] = fmaf(__uint_as_float(p[4 * q + 3]), sa * b.w, acc[4 * q + 3]);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[stage]);            // scales of this stage consumed
                pb ^= 1;
                if (++stage == PG_STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            const int64_t row = (int64_t)mb * PG_BM + row_in;
            const int64_t col0 = (int64_t)nb * PG_BN + half * 64;
            if (OUT_BF16) {
                uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(D) + row * ldd + col0);
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    dst[c] = make_uint4(pack_bf16(acc[8 * c], acc[8 * c + 1]), pack_bf16(acc[8 * c + 2], acc[8 * c + 3]),
                                        pack_bf16(acc[8 * c + 4], acc[8 * c + 5]),
                                        pack_bf16(acc[8 * c + 6], acc[8 * c + 7]));
            } else {
                float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(D) + row * ldd + col0);
#pragma unroll
                for (int c = 0; c < 16; ++c) dst[c] = make_float4(acc[4 * c], acc[4 * c + 1], acc[4 * c + 2], acc[4 * c + 3]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

int launch_gemm_pergroup(const uint8_t* A, const float* sa_t, const uint8_t* B, const float* sb_t, void* D,
                         int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, cudaStream_t st) {
    CUtensorMap ta, tb;
    if (!make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, A, M, K, 128, PG_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, B, N, K, 128, PG_BN, CU_TENSOR_MAP_SWIZZLE_128B))
        return MOSS_ERR_CUDA;
    const bool bf = d_dtype == MOSS_BF16;
    auto kern = bf ? gemm_pergroup_kernel<true> : gemm_pergroup_kernel<false>;
    static bool attr[2][kMaxDevices] = {};
    if (!smem_optin(kern, PgLayout::SMEM, attr[bf])) return MOSS_ERR_CUDA;
    const int64_t tiles = (M / PG_BM) * (N / PG_BN);
    const int grid = (int)std::min<int64_t>(tiles, sm_count());
    kern<<<grid, PG_THREADS, PgLayout::SMEM, st>>>(ta, tb, sa_t, sb_t, D, ldd, (int)M, (int)N, (int)K);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

}  // namespace moss
