// K2 v2: block-scaled MXFP8 GEMM on CTA pairs (tcgen05 cta_group::2).
//
//   D[m, n] = alpha * sum_k A[m,k] 2^(SFA[m,k/32]-127) B[n,k] 2^(SFB[n,k/32]-127),  alpha = (*sA)(*sB)
//
// Same contract as gemm.cu (reference gemm.py:115-129); this variant covers
// M % 256 == 0, N % 256 == 0, K % 128 == 0 (every Llama-7B fwd/dgrad/wgrad).
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A
// and half (128 rows) of B, so a pair moves 2 x 32 KB of operands per 128-K
// stage instead of the 2 x 48 KB two independent 128 x 256 CTAs would — the
// L2 -> SM traffic that bounds the 1-CTA kernel drops by a third.
//
// Roles (per CTA, 640 threads):
//   warp 0       TMA producer: 2-SM TMA loads of A/B (bytes credited to the
//                leader's full barrier), bulk copies of this CTA's SF
//   warp 1       leader only: MMA issuer (tcgen05.cp + tcgen05.mma cta_group::2,
//                multicast commits to both CTAs' empty / tmem_full barriers)
//   warp 2       TMEM allocator (cta_group::2)
//   warp 3       SF watcher: waits this CTA's SF bytes, then arrives on the
//                leader's full barrier (so the leader knows both SF halves landed)
//   warps 4-19   epilogue: 4 warps per TMEM lane quadrant, 64 columns each;
//                tcgen05.ld -> release TMEM to the leader -> alpha -> bf16/f32
//                -> 128B-swizzled smem -> TMA store (TMA reduce-add for accumulate)
#include <algorithm>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

constexpr int G2_BM = 128;       // rows per CTA (256 per pair)
constexpr int G2_BN = 256;       // columns per pair tile
constexpr int G2_BK = 128;
constexpr int G2_STAGES = 4;
constexpr int G2_EPI_WARPS = 16;
constexpr int G2_THREADS = (4 + G2_EPI_WARPS) * 32;

struct G2Layout {
    static constexpr int A_BYTES = G2_BM * G2_BK;              // 16 KB
    static constexpr int B_BYTES = (G2_BN / 2) * G2_BK;        // 16 KB (half of B per CTA)
    static constexpr int SFA_BYTES = 512;
    static constexpr int SFB_BYTES = (G2_BN / 128) * 512;      // full-N scales in each CTA
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + G2_STAGES * A_BYTES;
    static constexpr int OFF_SFA = OFF_B + G2_STAGES * B_BYTES;
    static constexpr int OFF_SFB = OFF_SFA + G2_STAGES * SFA_BYTES;
    static constexpr int OFF_UNIT = OFF_SFB + G2_STAGES * SFB_BYTES;
    static constexpr int OFF_STG = OFF_UNIT + SFB_BYTES;       // 16 x 4 KB epilogue staging
    static constexpr int OFF_BAR = OFF_STG + G2_EPI_WARPS * 4096;
    static constexpr int N_BARS = 3 * G2_STAGES + 2;          // full, sf_full, empty, tmem_full, tmem_empty
    static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
    static constexpr int SMEM = OFF_TMEM + 16 + 1024;
    static constexpr uint32_t TMEM_COLS = 512;                 // 256 accumulator + SF
};

template <bool OUT_BF16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(G2_THREADS, 1)
    gemm_mxf8_2cta_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmD, const uint8_t* __restrict__ sfa,
                          const uint8_t* __restrict__ sfb, const float* __restrict__ sA,
                          const float* __restrict__ sB, int M, int N, int K, int accumulate) {
    using L = G2Layout;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_a = smem + L::OFF_A;
    uint8_t* s_b = smem + L::OFF_B;
    uint8_t* s_sfa = smem + L::OFF_SFA;
    uint8_t* s_sfb = smem + L::OFF_SFB;
    uint8_t* s_unit = smem + L::OFF_UNIT;
    uint8_t* s_stg = smem + L::OFF_STG;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);   // leader's is the live one
    uint64_t* sf_full = full + G2_STAGES;
    uint64_t* empty = sf_full + G2_STAGES;
    uint64_t* tmem_full = empty + G2_STAGES;
    uint64_t* tmem_empty = tmem_full + 1;                              // leader's is the live one
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int m_pairs = M / (2 * G2_BM), n_tiles = N / G2_BN, num_tiles = m_pairs * n_tiles;
    const int kblocks = K / G2_BK;
    const bool unit_b = (sfb == nullptr);

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        prefetch_tmap(&tmD);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < G2_STAGES; ++s) {
            mbar_init(&full[s], 2);        // one SF-watcher arrival per CTA (+ A/B tx bytes of both)
            mbar_init(&sf_full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        mbar_init(tmem_empty, 2 * G2_EPI_WARPS);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_2cta(tmem_slot, L::TMEM_COLS);
    if (warp == 3 && unit_b) {
        for (int i = lane; i < L::SFB_BYTES / 4; i += 32) reinterpret_cast<uint32_t*>(s_unit)[i] = 0x7F7F7F7Fu;
        fence_proxy_async_smem();
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t tm_sfa = tmem + G2_BN;
    const uint32_t tm_sfb = tmem + G2_BN + 4;
    const uint32_t full_leader0 = mapa_shared(&full[0], 0);
    const uint32_t tmem_empty_leader = mapa_shared(tmem_empty, 0);

    if (warp == 0) {
        // ---------------- producer (both CTAs) ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            const uint32_t ab_bytes = L::A_BYTES + L::B_BYTES;
            const uint32_t sf_bytes = L::SFA_BYTES + (unit_b ? 0 : L::SFB_BYTES);
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                const int mp = tile % m_pairs, nt = tile / m_pairs;
                const int mb = mp * 2 + rank;                       // this CTA's 128-row block
                const int n0 = nt * G2_BN + rank * (G2_BN / 2);     // this CTA's half of B
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], 2 * ab_bytes);
                    const uint32_t fl = full_leader0 + stage * 8;
                    tma_load_2d_2sm(s_a + stage * L::A_BYTES, &tmA, fl, kb * G2_BK, mb * G2_BM);
                    tma_load_2d_2sm(s_b + stage * L::B_BYTES, &tmB, fl, kb * G2_BK, n0);
                    mbar_arrive_expect_tx(&sf_full[stage], sf_bytes);
                    bulk_load(s_sfa + stage * L::SFA_BYTES, sfa + ((int64_t)mb * kblocks + kb) * 512, 512,
                              &sf_full[stage]);
                    if (!unit_b) {
#pragma unroll
                        for (int j = 0; j < G2_BN / 128; ++j)
                            bulk_load(s_sfb + stage * L::SFB_BYTES + j * 512,
                                      sfb + ((int64_t)(nt * (G2_BN / 128) + j) * kblocks + kb) * 512, 512,
                                      &sf_full[stage]);
                    }
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 3) {
        // ---------------- SF watcher (both CTAs) ----------------
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&sf_full[stage], phase);
                    mbar_arrive_cluster(full_leader0 + stage * 8);
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer (leader CTA, one thread) ----------------
        if (leader && lane == 0) {
            if (unit_b) {
#pragma unroll
                for (int j = 0; j < G2_BN / 128; ++j)
                    tmem_cp_sf_2cta(tm_sfb + j * 4, umma_desc(smem_u32(s_unit + j * 512), 0, 128, kLayoutNone));
            }
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0;
            constexpr uint32_t idesc0 = mxf8_idesc(2 * G2_BM, G2_BN, 0, 0);
            for (int tile = pair; tile < num_tiles; tile += npairs) {
                mbar_wait(tmem_empty, acc_phase ^ 1);
                tc_fence_after();
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    tmem_cp_sf_2cta(tm_sfa, umma_desc(smem_u32(s_sfa + stage * L::SFA_BYTES), 0, 128, kLayoutNone));
                    if (!unit_b) {
#pragma unroll
                        for (int j = 0; j < G2_BN / 128; ++j)
                            tmem_cp_sf_2cta(tm_sfb + j * 4, umma_desc(smem_u32(s_sfb + stage * L::SFB_BYTES + j * 512),
                                                                      0, 128, kLayoutNone));
                    }
                    const uint64_t adesc = umma_desc(smem_u32(s_a + stage * L::A_BYTES), 0, 1024, kLayoutSW128);
                    const uint64_t bdesc = umma_desc(smem_u32(s_b + stage * L::B_BYTES), 0, 1024, kLayoutSW128);
#pragma unroll
                    for (int k = 0; k < G2_BK / 32; ++k)
                        mma_mxf8_2cta(tmem, adesc + 2 * k, bdesc + 2 * k, idesc0 | ((uint32_t)k << 29) | ((uint32_t)k << 4),
                                      tm_sfa, tm_sfb, (kb | k) != 0);
                    tc_commit_2cta_mc(&empty[stage], 0x3);
                    if (++stage == G2_STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                tc_commit_2cta_mc(tmem_full, 0x3);
                acc_phase ^= 1;
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs) ----------------
        const int ew = warp - 4;
        const int quad = warp & 3;            // TMEM lanes [32*quad, 32*quad+32)
        const int cq = ew >> 2;               // 64-column quarter
        uint8_t* stg = s_stg + ew * 4096;     // 32 rows x 128 B, SWIZZLE_128B
        const float alpha = __fmul_rn(*sA, *sB);
        uint32_t acc_phase = 0;
        for (int tile = pair; tile < num_tiles; tile += npairs) {
            const int mp = tile % m_pairs, nt = tile / m_pairs;
            const int row0 = (mp * 2 + rank) * G2_BM + quad * 32;
            const int col0 = nt * G2_BN + cq * 64;
            mbar_wait(tmem_full, acc_phase);
            tc_fence_after();
            uint32_t r[64];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + cq * 64;
            tmem_ld32(ta, *reinterpret_cast<uint32_t(*)[32]>(&r[0]));
            tmem_ld32(ta + 32, *reinterpret_cast<uint32_t(*)[32]>(&r[32]));
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tmem_empty_leader);   // accumulator may be overwritten now
            acc_phase ^= 1;
            if (OUT_BF16) {
                if (lane == 0) bulk_wait_read0();
                __syncwarp();
#pragma unroll
                for (int c = 0; c < 8; ++c) {
                    uint4 o;
                    o.x = pack_bf16(__uint_as_float(r[8 * c + 0]) * alpha, __uint_as_float(r[8 * c + 1]) * alpha);
                    o.y = pack_bf16(__uint_as_float(r[8 * c + 2]) * alpha, __uint_as_float(r[8 * c + 3]) * alpha);
                    o.z = pack_bf16(__uint_as_float(r[8 * c + 4]) * alpha, __uint_as_float(r[8 * c + 5]) * alpha);
                    o.w = pack_bf16(__uint_as_float(r[8 * c + 6]) * alpha, __uint_as_float(r[8 * c + 7]) * alpha);
                    *reinterpret_cast<uint4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = o;
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    tma_store_2d(&tmD, stg, col0, row0);
                    bulk_commit();
                }
            } else {
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 o = make_float4(__uint_as_float(r[32 * h + 4 * c + 0]) * alpha,
                                                     __uint_as_float(r[32 * h + 4 * c + 1]) * alpha,
                                                     __uint_as_float(r[32 * h + 4 * c + 2]) * alpha,
                                                     __uint_as_float(r[32 * h + 4 * c + 3]) * alpha);
                        *reinterpret_cast<float4*>(stg + lane * 128 + ((c ^ (lane & 7)) << 4)) = o;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (accumulate)
                            tma_reduce_add_2d(&tmD, stg, col0 + 32 * h, row0);
                        else
                            tma_store_2d(&tmD, stg, col0 + 32 * h, row0);
                        bulk_commit();
                    }
                }
            }
        }
        if (lane == 0) bulk_wait0();
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2cta(tmem, L::TMEM_COLS);
    }
}

template <bool OUT_BF16>
static int launch_gemm2_t(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                          const float* sB, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                          cudaStream_t st) {
    using L = G2Layout;
    auto kern = gemm_mxf8_2cta_kernel<OUT_BF16>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM) != cudaSuccess)
            return MOSS_ERR_CUDA;
        attr_set = true;
    }
    CUtensorMap ta, tb, td;
    if (!make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, A, M, K, 128, G2_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, B, N, K, 128, G2_BN / 2, CU_TENSOR_MAP_SWIZZLE_128B))
        return MOSS_ERR_CUDA;
    // D: [M, ldd] row-major; 32-row x 128 B boxes (64 bf16 or 32 f32 columns)
    {
        EncodeTiledFn enc = get_encode_fn();
        if (!enc) return MOSS_ERR_CUDA;
        const size_t esz = OUT_BF16 ? 2 : 4;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)(ldd * esz)};
        cuuint32_t box[2] = {(cuuint32_t)(128 / esz), 32u};
        cuuint32_t estr[2] = {1u, 1u};
        if (enc(&td, OUT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return MOSS_ERR_CUDA;
    }
    const int64_t tiles = (M / (2 * G2_BM)) * (N / G2_BN);
    const int pairs = (int)std::min<int64_t>(tiles, sm_count() / 2);
    kern<<<2 * pairs, G2_THREADS, L::SMEM, st>>>(ta, tb, td, SFA, SFB, sA, sB, (int)M, (int)N, (int)K, accumulate);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

// returns -1 when the shape is not covered by the pair kernel
int launch_gemm2(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                 const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                 cudaStream_t st) {
    if (M % (2 * G2_BM) || N % G2_BN || K % G2_BK) return -1;
    if ((reinterpret_cast<uintptr_t>(D) % 16) || (ldd * (d_dtype == MOSS_BF16 ? 2 : 4)) % 16) return -1;
    return d_dtype == MOSS_BF16 ? launch_gemm2_t<true>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, 0, st)
                                : launch_gemm2_t<false>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, accumulate, st);
}

}  // namespace moss
