// K2 v2: block-scaled MXFP8 GEMM on CTA pairs (tcgen05 cta_group::2).
//
//   D[m, n] = alpha * sum_k A[m,k] 2^(SFA[m,k/32]-127) B[n,k] 2^(SFB[n,k/32]-127),  alpha = (*sA)(*sB)
//
// Same contract as gemm.cu (reference gemm.py:115-129); this variant covers
// M % 256 == 0, N % 256 == 0, K % 128 == 0 (every Llama-7B fwd/dgrad/wgrad).
//
// A cluster of two CTAs on one TPC computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A
// and one half (128 rows) of B, so a pair moves 2 x 32 KB of operands per
// 128-K stage where two independent 128 x 256 CTAs move 2 x 48 KB.  The
// 1-CTA kernel is latency-bound on its 4 x 48 KB ring; the pair kernel keeps
// more stages in flight (32 KB + SF per stage) for the same FLOPs.
//
// Every load — A, B and both scale-factor operands — is a 2-SM TMA whose
// bytes are credited to the LEADER CTA's full barrier, so the MMA issuer
// waits on exactly one barrier per stage.
//
// Roles (per CTA, 640 threads):
//   warp 0       TMA producer (both CTAs)
//   warp 1       MMA issuer (leader CTA, one thread): tcgen05.cp + tcgen05.mma
//                cta_group::2, multicast commits to both CTAs' barriers
//   warp 2       TMEM allocator (cta_group::2)
//   warps 4-19   epilogue: 4 warps per TMEM lane quadrant, 64 columns each;
//                tcgen05.ld -> release TMEM (arrive on the leader) -> alpha ->
//                bf16/f32 -> global (direct stores, or swizzled smem + TMA store /
//                TMA reduce-add when TMA_EPI)
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

#ifdef G2_TIMELINE
// debug build only (tools/gemm_timeline.py): per pair, per tile, 6 globaltimer stamps
constexpr int G2_TL_TILES = 64;
__device__ unsigned long long g2_tl[74 * G2_TL_TILES * 8];
__device__ __forceinline__ unsigned long long g2_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define G2_STAMP(pair, it, ev)                                                            \
    do {                                                                                  \
        if ((pair) < 74 && (it) < G2_TL_TILES) g2_tl[((pair) * G2_TL_TILES + (it)) * 8 + (ev)] = g2_now(); \
    } while (0)
#else
#define G2_STAMP(pair, it, ev) \
    do {                       \
    } while (0)
#endif

constexpr int G2_BM = 128;       // rows per CTA (256 per pair)
constexpr int G2_BN = 256;       // columns per pair tile (the default; 128 with 2 accumulator stages)
constexpr int G2_BK = 128;

// BN = 256: one TMEM accumulator (256 columns + SF); BN = 128: two accumulator
// stages (2 x 128 columns) so the epilogue of tile i overlaps tile i+1's MMAs.
template <int STAGES, bool TMA_EPI, int EPI_WARPS, int BN>
struct G2Layout {
    static constexpr int ACC = BN == 128 ? 2 : 1;              // TMEM accumulator stages
    static constexpr int A_BYTES = G2_BM * G2_BK;              // 16 KB
    static constexpr int B_BYTES = (BN / 2) * G2_BK;           // half of B per CTA
    static constexpr int SFA_BYTES = 512;
    static constexpr int SFB_BYTES = (BN / 128) * 512;         // scales of all BN B rows in each CTA
    static constexpr int OFF_A = 0;
    static constexpr int OFF_B = OFF_A + STAGES * A_BYTES;
    static constexpr int OFF_SFA = OFF_B + STAGES * B_BYTES;
    static constexpr int OFF_SFB = OFF_SFA + STAGES * SFA_BYTES;
    static constexpr int OFF_UNIT = OFF_SFB + STAGES * SFB_BYTES;
    static constexpr int STG_BYTES = TMA_EPI ? 2048 : 0;       // per epilogue warp: 32 rows x 64 B
    static constexpr int OFF_STG = OFF_UNIT + SFB_BYTES;
    static constexpr int OFF_BAR = OFF_STG + EPI_WARPS * STG_BYTES;
    // full, empty, tmem_full[ACC], tmem_empty[ACC], split[EPI_WARPS] (tail-split partial loads)
    static constexpr int N_BARS = 2 * STAGES + 2 * ACC + EPI_WARPS;
    static constexpr int OFF_TMEM = OFF_BAR + N_BARS * 8;
    static constexpr int SMEM = OFF_TMEM + 16 + 1024;
    static constexpr uint32_t TMEM_COLS = 512;                 // ACC * BN = 256 accumulator + SF columns
};

// Tile raster: groups of |raster| m-pairs (raster > 0) walked n-major, or of
// |raster| n-tiles (raster < 0) walked m-major.  The ~74 concurrently running
// pair tiles then share one resident panel of the grouped operand (L2) while
// the other operand streams; the host (g2_raster) sizes the group so the
// resident panel fits the L2 budget and picks the orientation with the fewest
// DRAM bytes.  (A plain m-major walk re-read all of A for every n column on
// tall problems: 12288 x 4096 x 8192 ran at 49 % DRAM with 4x the bytes.)
__device__ __forceinline__ void g2_tile_coords(int tile, int m_pairs, int n_tiles, int raster, int& mp, int& nt) {
    if (raster > 0) {
        const int group = raster * n_tiles;
        const int gi = tile / group;
        const int first = gi * raster;
        const int gm = min(m_pairs - first, raster);
        const int r = tile - gi * group;
        mp = first + r % gm;
        nt = r / gm;
    } else {
        const int g = -raster;
        const int group = g * m_pairs;
        const int gi = tile / group;
        const int first = gi * g;
        const int gn = min(n_tiles - first, g);
        const int r = tile - gi * group;
        nt = first + r % gn;
        mp = r / gn;
    }
}

// Tail split (a 2-way stream-K of the last, partial wave; K >= 8192 only, see the
// launcher).  Units [0, split_first)
// are whole tiles; when the last wave holds rem <= npairs/2 tiles, each of them
// becomes two units over the two halves of K, both in the last wave on
// different pairs: role 1 (first half) hands its raw FP32 accumulator to role 2
// (second half) through a global workspace + per-warp flag, role 2 adds it and
// runs the normal epilogue.  The last wave then takes half a tile instead of a
// whole one (M = 4096 Llama-7B GEMMs: 256 tiles on 74 pairs = 3.46 waves).
struct G2Unit {
    int tile, kb0, kb1, role, slot;
};
__device__ __forceinline__ G2Unit g2_unit(int u, int split_first, int kblocks) {
    G2Unit w;
    if (u < split_first) {
        w.tile = u; w.kb0 = 0; w.kb1 = kblocks; w.role = 0; w.slot = 0;
    } else {
        const int v = u - split_first, h = v & 1, kh = kblocks >> 1;
        w.slot = v >> 1;
        w.tile = split_first + w.slot;
        w.kb0 = h ? kh : 0;
        w.kb1 = h ? kblocks : kh;
        w.role = 1 + h;
    }
    return w;
}

// SF buffers are viewed as [bytes/256, 256] u8 tensors: one 512 B chunk = box {256, 2}
__device__ __forceinline__ int sf_row_of_chunk(int64_t chunk) { return (int)(chunk * 2); }

// B_MN: B is stored [K, N] row-major (N contiguous: the weight W itself for
// dgrad, instead of a transposed copy); its tiles are loaded and described
// MN-major (UMMA SWIZZLE_128B MN-major canonical layout: 128-byte rows of N,
// 8-row K groups 1024 B apart), the instruction descriptor's b_major bit set.
template <bool OUT_BF16, int STAGES, bool TMA_EPI, int EPI_WARPS, int BN, bool B_MN = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__((4 + EPI_WARPS) * 32, 1)
    gemm_mxf8_2cta_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                          const __grid_constant__ CUtensorMap tmD, void* __restrict__ D, int64_t ldd,
                          const float* __restrict__ sA, const float* __restrict__ sB, int M, int N, int K,
                          int unit_b, int accumulate, int raster, uint32_t* __restrict__ d_amax,
                          int split_first, float4* __restrict__ sk_ws, uint32_t* __restrict__ sk_flags) {
    using L = G2Layout<STAGES, TMA_EPI, EPI_WARPS, BN>;
    constexpr int ACC = L::ACC;
    constexpr int COLS = BN / (EPI_WARPS / 4);      // accumulator columns per epilogue warp
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* s_a = smem + L::OFF_A;
    uint8_t* s_b = smem + L::OFF_B;
    uint8_t* s_sfa = smem + L::OFF_SFA;
    uint8_t* s_sfb = smem + L::OFF_SFB;
    uint8_t* s_unit = smem + L::OFF_UNIT;
    uint8_t* s_stg = smem + L::OFF_STG;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);   // the leader's are live
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;                              // [ACC]
    uint64_t* tmem_empty = tmem_full + ACC;                            // [ACC], the leader's are live
    uint64_t* split_bar = tmem_empty + ACC;                            // [EPI_WARPS]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L::OFF_TMEM);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x >> 1, npairs = gridDim.x >> 1;
    const int m_pairs = M / (2 * G2_BM), n_tiles = N / BN, num_tiles = m_pairs * n_tiles;
    const int kblocks = K / G2_BK;
    const int num_units = split_first + 2 * (num_tiles - split_first);

    if (warp == 0 && lane == 0 && cluster_ctarank() == 0) G2_STAMP(blockIdx.x >> 1, 1, 7);   // kernel entry
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        prefetch_tmap(&tmSFA);
        if (!unit_b) prefetch_tmap(&tmSFB);
        if (TMA_EPI) prefetch_tmap(&tmD);
    }
    if (warp == 1 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);        // leader's arrive.expect_tx; bytes from both CTAs
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < ACC; ++a) {
            mbar_init(&tmem_full[a], 1);
            mbar_init(&tmem_empty[a], 2 * EPI_WARPS);
        }
        for (int w = 0; w < EPI_WARPS; ++w) mbar_init(&split_bar[w], 1);
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
    // SF columns double-buffered by k-block parity: [256, 268) and [272, 284)
    const uint32_t tm_sfa = tmem + ACC * BN;
    const uint32_t tm_sfb = tmem + ACC * BN + 4;
    constexpr uint32_t SF_ALT = 16;

    if (warp == 0) {
        // ---------------- producer (both CTAs; warp-converged, one elected lane issues) ----------------
        const uint32_t full_leader0 = mapa_shared(&full[0], 0);
        const uint32_t cta_bytes = L::A_BYTES + L::B_BYTES + L::SFA_BYTES + (unit_b ? 0 : L::SFB_BYTES);
        int stage = 0;
        uint32_t phase = 0;
        for (int u = pair; u < num_units; u += npairs) {
            const G2Unit w = g2_unit(u, split_first, kblocks);
            int mp, nt;
            g2_tile_coords(w.tile, m_pairs, n_tiles, raster, mp, nt);
            const int mb = mp * 2 + rank;                       // this CTA's 128-row block of A
            const int n0 = nt * BN + rank * (BN / 2);           // this CTA's half of B
            for (int kb = w.kb0; kb < w.kb1; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                if (elect_one()) {
                    if (leader) mbar_arrive_expect_tx(&full[stage], 2 * cta_bytes);
                    const uint32_t fl = full_leader0 + stage * 8;
                    tma_load_2d_2sm(s_a + stage * L::A_BYTES, &tmA, fl, kb * G2_BK, mb * G2_BM);
                    if (B_MN)
                        tma_load_2d_2sm(s_b + stage * L::B_BYTES, &tmB, fl, n0, kb * G2_BK);
                    else
                        tma_load_2d_2sm(s_b + stage * L::B_BYTES, &tmB, fl, kb * G2_BK, n0);
                    tma_load_2d_2sm(s_sfa + stage * L::SFA_BYTES, &tmSFA, fl, 0,
                                    sf_row_of_chunk((int64_t)mb * kblocks + kb));
                    if (!unit_b) {
#pragma unroll
                        for (int j = 0; j < BN / 128; ++j)
                            tma_load_2d_2sm(s_sfb + stage * L::SFB_BYTES + j * 512, &tmSFB, fl, 0,
                                            sf_row_of_chunk((int64_t)(nt * (BN / 128) + j) * kblocks + kb));
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
        // ---------------- MMA issuer (leader CTA; warp-converged, one elected lane issues) ----------------
        if (leader) {
            if (unit_b) {
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < BN / 128; ++j) {
                        tmem_cp_sf_2cta(tm_sfb + j * 4, umma_desc(smem_u32(s_unit + j * 512), 0, 128, kLayoutNone));
                        tmem_cp_sf_2cta(tm_sfb + SF_ALT + j * 4,
                                        umma_desc(smem_u32(s_unit + j * 512), 0, 128, kLayoutNone));
                    }
                }
                __syncwarp();
            }
            int stage = 0;
            uint32_t phase = 0, acc_phase = 0, sfbuf = 0;   // acc_phase bit a: parity of accumulator stage a
            constexpr uint32_t idesc0 = mxf8_idesc(2 * G2_BM, BN, 0, 0) | (B_MN ? (1u << 16) : 0u);
            const uint64_t adesc0 = umma_desc(smem_u32(s_a), 0, 1024, kLayoutSW128);
            // MN-major: LBO = stride between 128-element N blocks (one block per CTA
            // at BN = 256: unused), SBO = 1024 B between 8-row K groups
            const uint64_t bdesc0 = umma_desc(smem_u32(s_b), B_MN ? L::B_BYTES : 0, 1024, kLayoutSW128);
            const uint64_t sfadesc0 = umma_desc(smem_u32(s_sfa), 0, 128, kLayoutNone);
            const uint64_t sfbdesc0 = umma_desc(smem_u32(s_sfb), 0, 128, kLayoutNone);
            auto copy_sf = [&](uint32_t sa, uint32_t sb) {
                tmem_cp_sf_2cta(sa, sfadesc0 + (uint64_t)((stage * L::SFA_BYTES) >> 4));
                if (!unit_b) {
#pragma unroll
                    for (int j = 0; j < BN / 128; ++j)
                        tmem_cp_sf_2cta(sb + j * 4, sfbdesc0 + (uint64_t)((stage * L::SFB_BYTES + j * 512) >> 4));
                }
            };
            int it_ = 0;
            for (int u = pair; u < num_units; u += npairs, ++it_) {
                const G2Unit w = g2_unit(u, split_first, kblocks);
                // The first k-block's scale factors go into TMEM BEFORE the accumulator
                // is released: the SF columns are separate and double-buffered, and
                // tcgen05 ops of this thread execute in issue order, so the copy cannot
                // overtake the previous tile's MMAs.  Takes the copies off the handoff.
                mbar_wait(&full[stage], phase);
                tc_fence_after();
                if (elect_one()) copy_sf(tm_sfa + sfbuf, tm_sfb + sfbuf);
                __syncwarp();
                const int acc = ACC == 1 ? 0 : (it_ & 1);
                mbar_wait(&tmem_empty[acc], ((acc_phase >> acc) & 1u) ^ 1u);
                tc_fence_after();
                if (lane == 0) G2_STAMP(pair, it_, 0);
                for (int kb = w.kb0; kb < w.kb1; ++kb) {
                    if (kb > w.kb0) {
                        mbar_wait(&full[stage], phase);
                        tc_fence_after();
                    }
                    if (elect_one()) {
                        const uint32_t sa = tm_sfa + sfbuf, sb = tm_sfb + sfbuf;
                        if (kb > w.kb0) copy_sf(sa, sb);
                        const uint64_t adesc = adesc0 + (uint64_t)((stage * L::A_BYTES) >> 4);
                        const uint64_t bdesc = bdesc0 + (uint64_t)((stage * L::B_BYTES) >> 4);
#pragma unroll
                        for (int k = 0; k < G2_BK / 32; ++k)
                            mma_mxf8_2cta(tmem + acc * BN, adesc + 2 * k, bdesc + (B_MN ? 256 * k : 2 * k),
                                          idesc0 | ((uint32_t)k << 29) | ((uint32_t)k << 4), sa, sb,
                                          ((kb - w.kb0) | k) != 0);
                        tc_commit_2cta_mc(&empty[stage], 0x3);
                    }
                    __syncwarp();
                    if (kb == w.kb0 && lane == 0) G2_STAMP(pair, it_, 1);
                    sfbuf ^= SF_ALT;
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                if (elect_one()) tc_commit_2cta_mc(&tmem_full[acc], 0x3);
                __syncwarp();
                if (lane == 0) G2_STAMP(pair, it_, 2);
                acc_phase ^= 1u << acc;
            }
        }
    } else if (warp >= 4) {
        // ---------------- epilogue (both CTAs) ----------------
        const int ew = warp - 4;
        const int quad = warp & 3;            // TMEM lanes [32*quad, 32*quad+32)
        const int cq = ew >> 2;               // column slice of the 256-column tile
        uint32_t tmem_empty_leader[ACC];
#pragma unroll
        for (int a = 0; a < ACC; ++a) tmem_empty_leader[a] = mapa_shared(&tmem_empty[a], 0);
        uint8_t* stg = s_stg + ew * L::STG_BYTES;
        const uint32_t stg_s = smem_u32(stg);
        const float alpha = __fmul_rn(*sA, *sB);
        // max |D| of the stored values (bf16: both halves of each packed word; f32: the
        // magnitude bits) for the quantizer that consumes D (producer-fused amax)
        uint32_t am = 0;
        uint32_t acc_phase = 0;
        int it_ = 0;
        for (int u = pair; u < num_units; u += npairs, ++it_) {
            const G2Unit w = g2_unit(u, split_first, kblocks);
            int mp, nt;
            g2_tile_coords(w.tile, m_pairs, n_tiles, raster, mp, nt);
            const int row0 = (mp * 2 + rank) * G2_BM + quad * 32;
            const int col0 = nt * BN + cq * COLS;
            const int acc = ACC == 1 ? 0 : (it_ & 1);
            mbar_wait(&tmem_full[acc], (acc_phase >> acc) & 1u);
            tc_fence_after();
            const bool stamp = ew == 0 && rank == 0 && lane == 0;
            if (stamp) G2_STAMP(pair, it_, 3);
            uint32_t r[COLS];
            const uint32_t ta = tmem + ((uint32_t)(quad * 32) << 16) + acc * BN + cq * COLS;
#pragma unroll
            for (int c = 0; c < COLS / 32; ++c) tmem_ld32(ta + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&r[32 * c]));
            tmem_ld_wait();
            if (stamp) G2_STAMP(pair, it_, 4);
            tc_fence_before();
            __syncwarp();
            // Accumulator may be overwritten now.  RELAXED arrive: nothing is handed
            // over through memory (tcgen05.wait::ld already has the values in
            // registers), and a release arrive waits ~1 us for this lane's
            // in-flight TMA stores of the previous tile (measured with the
            // G2_TIMELINE build: E5-E4 1.06 -> 0.10 us, the whole per-tile bubble).
            if (lane == 0)
                asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                                 tmem_empty_leader[acc])
                             : "memory");
            if (stamp) G2_STAMP(pair, it_, 5);
            acc_phase ^= 1u << acc;
            if (w.role) {
                // Tail split.  A split unit is its pair's LAST unit, so once the accumulator
                // is full every MMA has consumed its stage: the operand ring is free and
                // each epilogue warp stages its 32 rows x COLS partial (16 KB) there.  The
                // partial moves as ONE bulk copy per warp each way (the registers hold the
                // accumulator; per-thread loads would run 4 deep), thread-interleaved
                // float4s (c * 32 + lane): conflict-free smem, contiguous in global.
                static_assert(EPI_WARPS * 32 * COLS * 4 <= STAGES * (L::A_BYTES + L::B_BYTES), "partial staging");
                uint8_t* pst = smem + ew * (32 * COLS * 4);
                const uint32_t pst_s = smem_u32(pst);
                float4* part = sk_ws + ((size_t)w.slot * 2 * EPI_WARPS + rank * EPI_WARPS + ew) * (COLS / 4) * 32;
                uint32_t* flag = sk_flags + (w.slot * 2 * EPI_WARPS + rank * EPI_WARPS + ew);
                if (w.role == 1) {
#pragma unroll
                    for (int c = 0; c < COLS / 4; ++c)
                        sts128(pst_s + (c * 32 + lane) * 16, r[4 * c], r[4 * c + 1], r[4 * c + 2], r[4 * c + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        bulk_store(part, pst, 32 * COLS * 4);
                        bulk_commit();
                        bulk_wait0();                          // written, not just read from smem
                        asm volatile("fence.proxy.async.global;" ::: "memory");
                        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flag), "r"(1u) : "memory");
                    }
                    if (stamp) G2_STAMP(pair, it_, 6);
                    continue;                                  // role 2 stores the tile
                }
                if (lane == 0) {
                    uint32_t spins = 0;
                    while (ld_acquire_gpu_u32(flag) == 0u) {
                        if (++spins > (1u << 28)) __trap();
                    }
                    *flag = 0u;                                // ready for the next launch (stream-ordered)
                    asm volatile("fence.proxy.async.global;" ::: "memory");
                    mbar_arrive_expect_tx(&split_bar[ew], 32 * COLS * 4);
                    bulk_load(pst, part, 32 * COLS * 4, &split_bar[ew]);
                }
                __syncwarp();
                mbar_wait(&split_bar[ew], 0);                  // one use per launch: parity 0
                if (stamp) G2_STAMP(pair, it_, 6);
#pragma unroll
                for (int c = 0; c < COLS / 4; ++c) {
                    const uint4 q = lds128(pst_s + (c * 32 + lane) * 16);
                    r[4 * c] = __float_as_uint(__uint_as_float(r[4 * c]) + __uint_as_float(q.x));
                    r[4 * c + 1] = __float_as_uint(__uint_as_float(r[4 * c + 1]) + __uint_as_float(q.y));
                    r[4 * c + 2] = __float_as_uint(__uint_as_float(r[4 * c + 2]) + __uint_as_float(q.z));
                    r[4 * c + 3] = __float_as_uint(__uint_as_float(r[4 * c + 3]) + __uint_as_float(q.w));
                }
            }
            if (!TMA_EPI) {
                const int64_t row = row0 + lane;
                if (OUT_BF16) {
                    uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(D) + row * ldd + col0);
#pragma unroll
                    for (int c = 0; c < COLS / 8; ++c) {
                        uint4 o;
                        o.x = pack_bf16(__uint_as_float(r[8 * c + 0]) * alpha, __uint_as_float(r[8 * c + 1]) * alpha);
                        o.y = pack_bf16(__uint_as_float(r[8 * c + 2]) * alpha, __uint_as_float(r[8 * c + 3]) * alpha);
                        o.z = pack_bf16(__uint_as_float(r[8 * c + 4]) * alpha, __uint_as_float(r[8 * c + 5]) * alpha);
                        o.w = pack_bf16(__uint_as_float(r[8 * c + 6]) * alpha, __uint_as_float(r[8 * c + 7]) * alpha);
                        am = __vmaxu2(__vmaxu2(am, o.x & 0x7FFF7FFFu), o.y & 0x7FFF7FFFu);
                        am = __vmaxu2(__vmaxu2(am, o.z & 0x7FFF7FFFu), o.w & 0x7FFF7FFFu);
                        dst[c] = o;
                    }
                } else {
                    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(D) + row * ldd + col0);
#pragma unroll
                    for (int c = 0; c < COLS / 4; ++c) {
                        float4 o = make_float4(__uint_as_float(r[4 * c + 0]) * alpha, __uint_as_float(r[4 * c + 1]) * alpha,
                                               __uint_as_float(r[4 * c + 2]) * alpha, __uint_as_float(r[4 * c + 3]) * alpha);
                        if (accumulate) {
                            const float4 p = dst[c];
                            o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
                        }
                        am = max(max(am, __float_as_uint(o.x) & 0x7FFFFFFFu), __float_as_uint(o.y) & 0x7FFFFFFFu);
                        am = max(max(am, __float_as_uint(o.z) & 0x7FFFFFFFu), __float_as_uint(o.w) & 0x7FFFFFFFu);
                        dst[c] = o;
                    }
                }
            } else {
                // 32 rows x 64 B pieces, SWIZZLE_64B (16 B chunk ^ (row >> 1) & 3)
                constexpr int EPC = OUT_BF16 ? 32 : 16;          // elements per 64 B piece
                constexpr int NCH = COLS / EPC;
#pragma unroll
                for (int h = 0; h < NCH; ++h) {
                    if (lane == 0) bulk_wait_read0();
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        uint4 o;
                        if (OUT_BF16) {
                            const uint32_t* q = &r[32 * h + 8 * c];
                            o.x = pack_bf16(__uint_as_float(q[0]) * alpha, __uint_as_float(q[1]) * alpha);
                            o.y = pack_bf16(__uint_as_float(q[2]) * alpha, __uint_as_float(q[3]) * alpha);
                            o.z = pack_bf16(__uint_as_float(q[4]) * alpha, __uint_as_float(q[5]) * alpha);
                            o.w = pack_bf16(__uint_as_float(q[6]) * alpha, __uint_as_float(q[7]) * alpha);
                            am = __vmaxu2(__vmaxu2(am, o.x & 0x7FFF7FFFu), o.y & 0x7FFF7FFFu);
                            am = __vmaxu2(__vmaxu2(am, o.z & 0x7FFF7FFFu), o.w & 0x7FFF7FFFu);
                        } else {
                            const uint32_t* q = &r[16 * h + 4 * c];
                            o.x = __float_as_uint(__uint_as_float(q[0]) * alpha);
                            o.y = __float_as_uint(__uint_as_float(q[1]) * alpha);
                            o.z = __float_as_uint(__uint_as_float(q[2]) * alpha);
                            o.w = __float_as_uint(__uint_as_float(q[3]) * alpha);
                            am = max(max(am, o.x & 0x7FFFFFFFu), max(o.y & 0x7FFFFFFFu, o.z & 0x7FFFFFFFu));
                            am = max(am, o.w & 0x7FFFFFFFu);     // (d_amax is refused with accumulate)
                        }
                        sts128(stg_s + lane * 64 + ((c ^ ((lane >> 1) & 3)) << 4), o.x, o.y, o.z, o.w);
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int c0 = col0 + h * EPC;
                        if (!OUT_BF16 && accumulate)
                            tma_reduce_add_2d(&tmD, stg, c0, row0);
                        else
                            tma_store_2d(&tmD, stg, c0, row0);
                        bulk_commit();
                    }
                }
            }
        }
        if (TMA_EPI && lane == 0) bulk_wait0();
        if (ew == 0 && rank == 0 && lane == 0) G2_STAMP(pair, 0, 7);     // this pair's epilogue done
        if (d_amax) {
            // as f32 bits: |x| orders like its bits; NaN/Inf land at >= 0x7F800000 (flagged by the quantizer)
            uint32_t v = OUT_BF16 ? (max(am & 0xFFFFu, am >> 16) << 16) : am;
            v = __reduce_max_sync(0xFFFFFFFFu, v);
            if (lane == 0 && v) atomicMax(d_amax, v);
        }
    }
    tc_fence_before();
    cluster_sync_all();
    if (warp == 2) {
        tc_fence_after();
        tmem_dealloc_2cta(tmem, L::TMEM_COLS);
    }
}

// Raster choice (host): keep a panel of one operand L2-resident and stream the
// other.  Grouping m-pairs re-reads B once per group, grouping n-tiles re-reads
// A once per group; the group is the largest whose panel fits the budget
// (MOSS_GEMM2_L2MB, default 80 MB of the 126 MB L2) and the orientation with
// the fewer modelled DRAM bytes wins.  Measured over the 12 LayerStack GEMMs
// (ncu dram bytes per launch): fixed 8-m-pair groups (MOSS_GEMM2_L2MB=0) 437 MB,
// budget 40 -> 376, 80 -> 366, 120 -> 514 (the panel no longer survives a wave
// of streamed tiles), every launch at 80 at or below the fixed raster.  A
// budget that also charges one wave of streamed panels was tried and was worse
// (430 MB: it falls back to tiny groups on K = 22016 where concurrent tiles
// still share panels within a wave).
static int g2_raster(int64_t m_pairs, int64_t n_tiles, int BN, int64_t K) {
    static int64_t budget = -1;
    if (budget < 0) {
        const char* e = getenv("MOSS_GEMM2_L2MB");
        budget = (e ? atoll(e) : 80) << 20;
    }
    if (budget == 0) return 8;
    const int64_t a_pair = 2 * G2_BM * K, b_tile = (int64_t)BN * K;       // one panel (all of K)
    const int64_t gm = std::max<int64_t>(1, std::min<int64_t>(m_pairs, budget / a_pair));
    const int64_t gn = std::max<int64_t>(1, std::min<int64_t>(n_tiles, budget / b_tile));
    const int64_t bytes_m = m_pairs * a_pair + ((m_pairs + gm - 1) / gm) * n_tiles * b_tile;
    const int64_t bytes_n = n_tiles * b_tile + ((n_tiles + gn - 1) / gn) * m_pairs * a_pair;
    return bytes_m <= bytes_n ? (int)gm : -(int)gn;
}

// Tail-split workspace (per device; allocated on first use outside stream
// capture, flags zeroed once and re-zeroed by their consumers).  Split GEMMs
// on two streams of one device at the same time would share it: every MOSS
// GEMM of a training step runs on the compute stream.
constexpr int G2_SK_SLOTS = 64;                   // split tiles per launch (<= npairs / 2)
struct G2SplitWs {
    float4* part = nullptr;
    uint32_t* flags = nullptr;
};
static bool g2_split_ws(cudaStream_t st, G2SplitWs& out) {
    static G2SplitWs ws[kMaxDevices];
    G2SplitWs& w = ws[current_device()];
    if (!w.part) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return false;
        void *p = nullptr, *f = nullptr;
        if (cudaMalloc(&p, (size_t)G2_SK_SLOTS * 256 * 256 * sizeof(float)) != cudaSuccess) return false;
        if (cudaMalloc(&f, (size_t)G2_SK_SLOTS * 32 * sizeof(uint32_t)) != cudaSuccess ||
            cudaMemset(f, 0, (size_t)G2_SK_SLOTS * 32 * sizeof(uint32_t)) != cudaSuccess ||
            cudaDeviceSynchronize() != cudaSuccess) {
            cudaFree(p);
            return false;
        }
        w.part = reinterpret_cast<float4*>(p);
        w.flags = reinterpret_cast<uint32_t*>(f);
    }
    out = w;
    return true;
}

// MOSS_GEMM2_SPLIT=0 disables the tail split (A/B on the box)
static int g2_split_enabled() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_GEMM2_SPLIT");
        v = e ? (e[0] != '0') : 1;
    }
    return v;
}

template <bool OUT_BF16, int STAGES, bool TMA_EPI, int EPI_WARPS, int BN = 256, bool B_MN = false>
static int launch_gemm2_t(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                          const float* sB, void* D, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                          float* d_amax, cudaStream_t st) {
    using L = G2Layout<STAGES, TMA_EPI, EPI_WARPS, BN>;
    auto kern = gemm_mxf8_2cta_kernel<OUT_BF16, STAGES, TMA_EPI, EPI_WARPS, BN, B_MN>;
    static bool attr_set[kMaxDevices] = {};
    if (!smem_optin(kern, L::SMEM, attr_set)) return MOSS_ERR_CUDA;
    CUtensorMap ta, tb, tsa, tsb, td;
    const int64_t sfa_rows = ((M + 127) / 128) * (K / 128) * 2;
    const int64_t sfb_rows = ((N + 127) / 128) * (K / 128) * 2;
    if (!make_tmap_2d(&ta, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, A, M, K, 128, G2_BM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !(B_MN ? make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, B, K, N, BN / 2, G2_BK, CU_TENSOR_MAP_SWIZZLE_128B)
               : make_tmap_2d(&tb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, B, N, K, 128, BN / 2, CU_TENSOR_MAP_SWIZZLE_128B)) ||
        !make_tmap_2d(&tsa, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, SFA, sfa_rows, 256, 256, 2, CU_TENSOR_MAP_SWIZZLE_NONE))
        return MOSS_ERR_CUDA;
    tsb = tsa;
    if (SFB && !make_tmap_2d(&tsb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, SFB, sfb_rows, 256, 256, 2,
                             CU_TENSOR_MAP_SWIZZLE_NONE))
        return MOSS_ERR_CUDA;
    td = ta;
    if (TMA_EPI) {
        EncodeTiledFn enc = get_encode_fn();
        if (!enc) return MOSS_ERR_CUDA;
        const size_t esz = OUT_BF16 ? 2 : 4;
        cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
        cuuint64_t strides[1] = {(cuuint64_t)(ldd * esz)};
        cuuint32_t box[2] = {(cuuint32_t)(64 / esz), 32u};
        cuuint32_t estr[2] = {1u, 1u};
        if (enc(&td, OUT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, D, dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return MOSS_ERR_CUDA;
    }
    const int64_t tiles = (M / (2 * G2_BM)) * (N / BN);
    const int pairs = (int)std::min<int64_t>(tiles, sm_count() / 2);
    const int raster = g2_raster(M / (2 * G2_BM), N / BN, BN, K);
    // tail split when the last wave is at most half full (2 units per tail tile fit one wave)
    int split_first = (int)tiles;
    G2SplitWs sk;
    const int64_t rem = tiles % pairs;
    // (the partial exchange costs ~4-6 us at the end of the kernel — measured with the
    // G2_TIMELINE build, tools/gemm_split_timeline.py — so it pays only when half a
    // tile is longer than that: K >= 8192, a 256 x 256 x 8192 tile is ~26 us)
    if (BN == 256 && rem > 0 && 2 * rem <= pairs && rem <= G2_SK_SLOTS && K >= 8192 &&
        g2_split_enabled() && g2_split_ws(st, sk))
        split_first = (int)(tiles - rem);
    if (d_amax && zero_word(d_amax, st) != cudaSuccess) return MOSS_ERR_CUDA;
    kern<<<2 * pairs, (4 + EPI_WARPS) * 32, L::SMEM, st>>>(ta, tb, tsa, tsb, td, D, ldd, sA, sB, (int)M, (int)N, (int)K,
                                                 SFB == nullptr, accumulate, raster,
                                                 reinterpret_cast<uint32_t*>(d_amax), split_first,
                                                 sk.part, sk.flags);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

// MOSS_GEMM2_MODE (A/B testing on B200):
//   2 (default) 256 x 256 pair tiles, 1 TMEM accumulator, 6 stages, 8 epilogue warps, TMA-store epilogue
//   3           256 x 128 pair tiles, 2 TMEM accumulator stages (epilogue overlapped), 8 stages
static int gemm2_mode() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_GEMM2_MODE");
        v = e ? (e[0] - '0') : 2;
        if (v != 2 && v != 3) v = 2;
    }
    return v;
}

// returns -1 when the shape is not covered by the pair kernel
int launch_gemm2(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                 const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                 float* d_amax, cudaStream_t st) {
    if (M % (2 * G2_BM) || N % 128 || K % G2_BK) return -1;
    if ((reinterpret_cast<uintptr_t>(D) % 16) || (ldd * (d_dtype == MOSS_BF16 ? 2 : 4)) % 16) return -1;
    const bool bf = d_dtype == MOSS_BF16;
    const bool n128 = gemm2_mode() == 3 || N % G2_BN != 0;
    if (n128)
        return bf ? launch_gemm2_t<true, 8, true, 8, 128>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, 0, d_amax, st)
                  : launch_gemm2_t<false, 8, true, 8, 128>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, accumulate, d_amax, st);
    return bf ? launch_gemm2_t<true, 6, true, 8>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, 0, d_amax, st)
              : launch_gemm2_t<false, 6, true, 8>(A, SFA, B, SFB, sA, sB, D, ldd, M, N, K, accumulate, d_amax, st);
}

// dgrad with the weight as stored: B = W [K, N] row-major, per-tensor (unit SF)
int launch_gemm2_bkn(const uint8_t* A, const uint8_t* SFA, const uint8_t* B_kn, const float* sA, const float* sB,
                     void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, float* d_amax,
                     cudaStream_t st) {
    if (M % (2 * G2_BM) || N % G2_BN || K % G2_BK) return MOSS_ERR_SHAPE;
    if ((reinterpret_cast<uintptr_t>(D) % 16) || (ldd * (d_dtype == MOSS_BF16 ? 2 : 4)) % 16) return MOSS_ERR_ALIGN;
    return d_dtype == MOSS_BF16
               ? launch_gemm2_t<true, 6, true, 8, 256, true>(A, SFA, B_kn, nullptr, sA, sB, D, ldd, M, N, K, 0, d_amax, st)
               : launch_gemm2_t<false, 6, true, 8, 256, true>(A, SFA, B_kn, nullptr, sA, sB, D, ldd, M, N, K, 0, d_amax, st);
}

}  // namespace moss

#ifdef G2_TIMELINE
extern "C" int moss_g2_timeline(void* host_dst) {
    return cudaMemcpyFromSymbol(host_dst, moss::g2_tl, sizeof(moss::g2_tl)) == cudaSuccess ? 0 : 5;
}
#endif
