// K2: block-scaled MXFP8 GEMM on sm_100a tensor cores.
//
//   D[m, n] = alpha * sum_k A[m,k] * 2^(SFA[m,k/32]-127) * B[n,k] * 2^(SFB[n,k/32]-127)
//   alpha   = (*sA) * (*sB)     (the two FP32 global scales, applied once in the epilogue)
//
// This is the dataflow of gemm_mx_epilogue (reference gemm.py:115-129): the
// per-32 block scales are applied by the tensor core itself
// (tcgen05.mma ... kind::mxf8f6f4.block_scale, E8M0 scales in TMEM), the
// global scales once per output.  No dequantisation or partial-sum fix-up
// runs in the K loop.
//
// Structure (one CTA per SM, persistent over 128 x BN output tiles):
//   warp 0      TMA producer: A/B tiles (128B-swizzled) + SF chunks (bulk copies)
//   warp 1      MMA issuer: tcgen05.cp SF smem->TMEM, 4 x tcgen05.mma per 128-K stage
//   warp 2      TMEM allocator
//   warps 4-11  epilogue: tcgen05.ld -> *alpha -> bf16/f32 -> global
// Pipelines: STAGES-deep smem ring (full/empty mbarriers), one TMEM
// accumulator (tmem_full/tmem_empty mbarriers).
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

constexpr int G_BM = 128;
constexpr int G_BK = 128;
constexpr int G_THREADS = 384;
constexpr int G_EPI_WARPS = 8;

template <int BN, int STAGES>
struct GemmLayout {
    static constexpr int A_BYTES = G_BM * G_BK;            // 16 KB
    static constexpr int B_BYTES = BN * G_BK;              // 16/32 KB
    static constexpr int SFB_BYTES = (BN / 128) * 512;
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
    static constexpr int OFF_SFA = OFF_B + STAGES * B_BYTES;
    static constexpr int OFF_SFB = OFF_SFA + STAGES * 512;
    static constexpr int OFF_UNIT = OFF_SFB + STAGES * SFB_BYTES;
    static constexpr int OFF_BAR = OFF_UNIT + SFB_BYTES;
    static constexpr int N_BARS = 2 * STAGES + 2;
    static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
    static constexpr int BYTES = OFF_TMEM + 16;
    static constexpr int SMEM = BYTES + 1024;  // slack for 1 KB alignment
    static constexpr uint32_t TMEM_COLS = (BN + 12) <= 256 ? 256 : 512;
};

template <int BN, int STAGES, bool OUT_BF16>
__global__ void __launch_bounds__(G_THREADS, 1)
    gemm_mxf8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const uint8_t* __restrict__ sfa, const uint8_t* __restrict__ sfb, const float* __restrict__ sA,
                     const float* __restrict__ sB, void* __restrict__ D, int64_t ldd, int M, int N, int K,
                     int accumulate) {
    using L = GemmLayout<BN, STAGES>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_a = smem + L::OFF_A;
    uint8_t* s_b = smem + L::OFF_B;
    uint8_t* s_sfa = smem + L::OFF_SFA;
    uint8_t* s_sfb = smem + L::OFF_SFB;
    uint8_t* s_unit = smem + L::OFF_UNIT;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint64_t* tmem_empty = tmem_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m_tiles = M / G_BM, n_tiles = N / BN, num_tiles = m_tiles * n_tiles;
    const int kblocks = K / G_BK;
    const bool unit_b = (sfb == nullptr);

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, G_EPI_WARPS);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, L::TMEM_COLS);
    if (warp == 3 && unit_b) {
        for (int i = lane; i < L::SFB_BYTES / 4; i += 32) reinterpret_cast<uint32_t*>(s_unit)[i] = 0x7F7F7F7Fu;
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_acc = tmem;
    const uint32_t tm_sfa = tmem + BN;
    const uint32_t tm_sfb = tmem + BN + 4;

    if (warp == 0) {
        // ---------------- TMA producer (warp-converged, one elected lane issues) ----------------
        int stage = 0;
        uint32_t phase = 0;
        const uint32_t bytes = L::A_BYTES + L::B_BYTES + 512 + (unit_b ? 0 : L::SFB_BYTES);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mb = tile % m_tiles, nb = tile / m_tiles;
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&full[stage], bytes);
                    tma_load_2d(s_a + stage * L::A_BYTES, &tmA, &full[stage], kb * G_BK, mb * G_BM);
                    tma_load_2d(s_b + stage * L::B_BYTES, &tmB, &full[stage], kb * G_BK, nb * BN);
                    bulk_load(s_sfa + stage * 512, sfa + ((int64_t)mb * kblocks + kb) * 512, 512, &full[stage]);
                    if (!unit_b) {
#pragma unroll
                        for (int j = 0; j < BN / 128; ++j)
                            bulk_load(s_sfb + stage * L::SFB_BYTES + j * 512,
                                      sfb + ((int64_t)(nb * (BN / 128) + j) * kblocks + kb) * 512, 512, &full[stage]);
                    }
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (warp-converged, one elected lane issues) ----------------
        if (unit_b) {
            if (elect_one()) {
#pragma unroll
                for (int j = 0; j < BN / 128; ++j)
                    tmem_cp_sf(tm_sfb + j * 4, umma_desc(smem_u32(s_unit + j * 512), 0, 128, kLayoutNone));
            }
            __syncwarp();
        }
        int stage = 0;
        uint32_t phase = 0, acc_phase = 0;
        const uint64_t adesc0 = umma_desc(smem_u32(s_a), 0, 1024, kLayoutSW128);
        const uint64_t bdesc0 = umma_desc(smem_u32(s_b), 0, 1024, kLayoutSW128);
        const uint64_t sfadesc0 = umma_desc(smem_u32(s_sfa), 0, 128, kLayoutNone);
        const uint64_t sfbdesc0 = umma_desc(smem_u32(s_sfb), 0, 128, kLayoutNone);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            mbar_wait(tmem_empty, acc_phase ^ 1);
            tc_fence_after();
            for (int kb = 0; kb < kblocks; ++kb) {
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) {
                    tmem_cp_sf(tm_sfa, sfadesc0 + (uint64_t)((stage * 512) >> 4));
                    if (!unit_b) {
#pragma unroll
                        for (int j = 0; j < BN / 128; ++j)
                            tmem_cp_sf(tm_sfb + j * 4, sfbdesc0 + (uint64_t)((stage * L::SFB_BYTES + j * 512) >> 4));
                    }
                    const uint64_t adesc = adesc0 + (uint64_t)((stage * L::A_BYTES) >> 4);
                    const uint64_t bdesc = bdesc0 + (uint64_t)((stage * L::B_BYTES) >> 4);
#pragma unroll
                    for (int k = 0; k < G_BK / 32; ++k)
                        mma_mxf8(tm_acc, adesc + 2 * k, bdesc + 2 * k, mxf8_idesc(G_BM, BN, k, k), tm_sfa, tm_sfb,
                                 (kb | k) != 0);
                    tc_commit(&empty[stage]);
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (elect_one()) tc_commit(tmem_full);
            __syncwarp();
            acc_phase ^= 1;
        }
    } else if (warp >= 4) {
        // ---------------- epilogue ----------------
        const int ew = warp - 4;
        const int quad = warp & 3;          // TMEM lane quadrant this warp may access
        const int half = ew >> 2;           // which half of the BN columns
        const float alpha = __fmul_rn(*sA, *sB);
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int mb = tile % m_tiles, nb = tile / m_tiles;
            mbar_wait(tmem_full, acc_phase);
            tc_fence_after();
            const int64_t row = (int64_t)mb * G_BM + quad * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 2 / 32; ++c) {
                const int ct = half * (BN / 2) + c * 32;
                uint32_t r[32];
                tmem_ld32(tm_acc + ((uint32_t)(quad * 32) << 16) + ct, r);
                tmem_ld_wait();
                const int64_t col = (int64_t)nb * BN + ct;
                if (OUT_BF16) {
                    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(D) + row * ldd + col);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        uint4 o;
                        o.x = pack_bf16(__uint_as_float(r[8 * q + 0]) * alpha, __uint_as_float(r[8 * q + 1]) * alpha);
                        o.y = pack_bf16(__uint_as_float(r[8 * q + 2]) * alpha, __uint_as_float(r[8 * q + 3]) * alpha);
                        o.z = pack_bf16(__uint_as_float(r[8 * q + 4]) * alpha, __uint_as_float(r[8 * q + 5]) * alpha);
                        o.w = pack_bf16(__uint_as_float(r[8 * q + 6]) * alpha, __uint_as_float(r[8 * q + 7]) * alpha);
                        dst[q] = o;
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(D) + row * ldd + col);
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        float4 o = make_float4(__uint_as_float(r[4 * q + 0]) * alpha, __uint_as_float(r[4 * q + 1]) * alpha,
                                               __uint_as_float(r[4 * q + 2]) * alpha, __uint_as_float(r[4 * q + 3]) * alpha);
                        if (accumulate) {
                            const float4 p = dst[q];
                            o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
                        }
                        dst[q] = o;
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(tmem_empty);
            acc_phase ^= 1;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc(tmem, L::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ host side
// K-major uint8 operand [rows, k]: box = 128 B of K x box_rows rows, 128B swizzle.
static bool make_kmajor_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t k, int box_rows) {
    return make_tmap_2d(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, ptr, rows, k, 128, box_rows, CU_TENSOR_MAP_SWIZZLE_128B);
}

template <int BN, int STAGES, bool OUT_BF16>
static int launch_gemm_t(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                         const float* sB, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                         cudaStream_t st) {
    using L = GemmLayout<BN, STAGES>;
    auto kern = gemm_mxf8_kernel<BN, STAGES, OUT_BF16>;
    static bool attr_set[kMaxDevices] = {};
    if (!smem_optin(kern, L::SMEM, attr_set)) return MOSS_ERR_CUDA;
    CUtensorMap ta, tb;
    if (!make_kmajor_map(&ta, A, M, K, G_BM) || !make_kmajor_map(&tb, B, N, K, BN)) return MOSS_ERR_CUDA;
    const int sms = sm_count();
    const int64_t tiles = (M / G_BM) * (N / BN);
    const int grid = (int)std::min<int64_t>(tiles, sms);
    kern<<<grid, G_THREADS, L::SMEM, st>>>(ta, tb, SFA, SFB, sA, sB, D, ldd, (int)M, (int)N, (int)K, accumulate);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

int launch_gemm2(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                 const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                 float* d_amax, cudaStream_t st);
int launch_amax(const void* x, int dtype, int64_t n, float* amax, uint32_t* flags, cudaStream_t st);

static int gemm_variant() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_GEMM_VARIANT");   // "1" forces the 1-CTA kernel (A/B testing)
        v = (e && e[0] == '1') ? 1 : 2;
    }
    return v;
}

int launch_gemm(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                float* d_amax, uint32_t* flags, cudaStream_t st) {
    if (gemm_variant() == 2) {
        const int r = launch_gemm2(A, SFA, B, SFB, sA, sB, D, d_dtype, ldd, M, N, K, accumulate, d_amax, st);
        if (r >= 0) return r;
    }
    const bool bn256 = (N % 256) == 0;
    int r;
    if (d_dtype == MOSS_BF16)
        r = bn256 ? launch_gemm_t<256, 4, true>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, 0, st)
                  : launch_gemm_t<128, 6, true>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, 0, st);
    else
        r = bn256 ? launch_gemm_t<256, 4, false>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, accumulate, st)
                  : launch_gemm_t<128, 6, false>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, accumulate, st);
    // the 1-CTA kernel has no amax epilogue: a separate pass over D (contiguous D only, checked by the caller)
    if (r == MOSS_OK && d_amax) r = launch_amax(D, d_dtype, M * N, d_amax, flags, st);
    return r;
}

}  // namespace moss
