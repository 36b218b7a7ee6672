// K1 v4: single-launch two-level MOSS quantizer for bf16 tensors whose sides
// are multiples of 128 — the global amax, the per-32 E8M0 scales and the E4M3
// codes (row-wise and/or column-wise) in ONE kernel.
//
// Semantics: quant_two_level (reference quantize.py:127-173); the column-wise
// output is quant_two_level(x.T) with x's global scale.
//
// Dataflow (2 CTAs of 256 threads per SM, each a 3-slot ring of 128 x 128 bf16 tiles):
//   phase A  (skipped when the producer supplies amax)  TMA-stream the CTA's
//            tiles and reduce max|x|; the last 3 tiles stay resident in smem.
//   barrier  one grid-wide arrive/release on a caller-owned workspace word;
//            every CTA then reads the tensor amax (g = amax/448).
//   phase B  quantize the resident tiles first, then the rest in DESCENDING
//            order, i.e. most recently read (L2-hot) first.  Row and column
//            passes read the tile into registers (the column pass with
//            ldmatrix.trans), the codes are written back INTO the same slot
//            (TMA SWIZZLE_128B layout) and TMA-stored; the slot is reloaded
//            once the store has read it.  Producer mode on big tensors takes
//            the last quarter of its tiles from a global counter (load balance).
//
// Arithmetic per element (FFMA2/FMUL2 pairs, sm_100):
//   z = RN(x / eff) = q0 - r*(eff*q0 - x), q0 = RN(x*r), r = RN(1/eff)
//   with r = RN(1/g) * 2^-e exact (eff = g*2^e, normal).  This 3-op division
//   equals IEEE div.rn.f32 for EVERY bf16 dividend and every f32 divisor
//   significand when r is the correctly rounded reciprocal: exhaustively
//   checked over 2^23 x 256 significand pairs (tests/test_division_proof.py).
//   s_i = RN(bmax/448) uses the same sequence with r = RN(1/448).
//   e_i = ceil(log2(s_i/g)) = (bits(s_i) - bits(g) + 0x7FFFFF) >> 23 for
//   normal s_i, g (exact integer form of fp8.py:205-208).
// A warp with any block outside that fast window (eff beyond [2^-60, 2^60):
// late-training gradients, tiny blocks) takes the general path: the same
// division on power-of-two-rescaled operands (q4_encode), exact for every
// positive finite eff; only eff = 0 / non-finite falls back to IEEE div.rn.
#include <algorithm>

#include "common.cuh"
#include "host_utils.cuh"

namespace moss {

constexpr int Q4_T = 128;
constexpr int Q4_IN = Q4_T * Q4_T * 2;     // 32 KB bf16 tile
constexpr int Q4_S = 3;                    // slots per CTA
constexpr int Q4_THREADS = 256;
constexpr int Q4_SMEM = Q4_S * Q4_IN + 2 * 1024 + 64 + 1024;   // slots, 2 x SF staging, barriers, align

#ifdef Q4_TIMELINE
// debug build only (tools/k1_timeline.py): per CTA of the LAST launch, globaltimer /
// clock64 at entry, after the first tile arrived, at exit; SM id; tiles processed
__device__ unsigned long long q4_tl[1024 * 8];
#endif

// workspace words (caller-owned, zero-initialised once; one stream at a time)
constexpr int WS_ARRIVE = 0, WS_GEN = 1, WS_AMAX0 = 2;   // amax slots [2], [3] by generation parity
constexpr int WS_TILE = 4, WS_DONE = 5;                  // producer mode: dynamic tile counter, CTAs done

__device__ __forceinline__ uint32_t q4_in_off(int r, int c) {   // bf16 tile, two 64-col SWIZZLE_128B boxes
    return (uint32_t)((c >> 6) * 16384 + r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4) + ((c & 7) << 1));
}
__device__ __forceinline__ uint32_t q4_out_off(int r, int byte) {   // u8 128x128 tile, SWIZZLE_128B
    return (uint32_t)(r * 128 + ((((byte >> 4) & 7) ^ (r & 7)) << 4) + (byte & 15));
}
__device__ __forceinline__ int q4_sf_in_chunk(int r, int kb) { return ((r & 31) << 4) + ((r >> 5) << 2) + kb; }

// ---- packed f32x2 arithmetic (FMUL2 / FFMA2)
__device__ __forceinline__ uint64_t pk(float lo, float hi) {
    uint64_t d;
    asm("mov.b64 %0, {%1, %2};" : "=l"(d) : "f"(lo), "f"(hi));
    return d;
}
__device__ __forceinline__ void upk(uint64_t d, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(d));
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
    uint64_t d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
    uint64_t d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
// RN(x / b) for a pair given xn = -x, nr = -RN(1/b), b normal (see header):
//   q0 = RN(x r), rem = RN(b q0 - x) (exact), q = RN(q0 - r rem).
// Working on -x keeps the sign of zero: x = -0 gives q = -0 (code 0x80).
__device__ __forceinline__ uint64_t div2n(uint64_t xn, uint64_t b, uint64_t nr) {
    const uint64_t q0 = fmul2(xn, nr);
    const uint64_t rem = ffma2(b, q0, xn);
    return ffma2(nr, rem, q0);
}
__device__ __forceinline__ float div1(float x, float nb, float r) {
    const float q0 = __fmul_rn(x, r);
    return __fmaf_rn(r, __fmaf_rn(nb, q0, x), q0);
}

struct Q4Global {
    float g;         // global scale f32(amax/448), 0 -> 1
    uint32_t gbits;
    float rg;        // RN(1/g) (valid when g_normal)
    bool g_normal;
    bool fast;       // g normal and in [2^-60, 2^60): the block fast path applies
    int emin;        // fast path needs e in [emin, emax]: eff = g 2^e in [2^-60, 2^60), e in [-127, 127]
    uint32_t erange; // emax - emin
};

__device__ __forceinline__ Q4Global q4_global(float amax) {
    Q4Global G;
    G.g = global_scale_from_amax(amax);
    G.gbits = __float_as_uint(G.g);
    G.g_normal = G.gbits >= 0x00800000u;
    G.rg = __frcp_rn(G.g);
    const int eg = (int)(G.gbits >> 23);
    G.fast = G.g_normal && eg >= 67 && eg <= 186;
    G.emin = max(67 - eg, -127);
    G.erange = (uint32_t)(min(186 - eg, 127) - G.emin);
    return G;
}

// Unpack NP packed bf16 pairs (element 2i = low half) into NEGATED floats:
// -lo = (w << 16) ^ 0x80000000, -hi = (w & 0xFFFF0000) ^ 0x80000000 (the
// negations fold into the FMUL2/FFMA2 operands).  Returns max |x|.
// (Moving the hi unpack to two IMADs on the FMA pipe measured 12 % slower.)
template <int NP>
__device__ __forceinline__ float q4_unpack(const uint32_t (&w)[NP], float (&lo)[NP], float (&hi)[NP]) {
#pragma unroll
    for (int i = 0; i < NP; ++i) {
        lo[i] = __uint_as_float(w[i] * 65536u + 0x80000000u);
        hi[i] = __uint_as_float((w[i] & 0xFFFF0000u) ^ 0x80000000u);
    }
    // block max |x| on the packed words: one max.xorsign.abs.bf16x2 per pair of
    // words (magnitude = max(|a|, |b|) per half, exact; the sign bit is masked)
    uint32_t t[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) t[i] = w[i];
#pragma unroll
    for (int step = 1; step < NP; step *= 2) {
#pragma unroll
        for (int i = 0; i + step < NP; i += 2 * step)
            asm("max.xorsign.abs.bf16x2 %0, %1, %2;" : "=r"(t[i]) : "r"(t[i]), "r"(t[i + step]));
    }
    const uint32_t mm = t[0] & 0x7FFF7FFFu;
    return fmaxf(__uint_as_float(mm << 16), __uint_as_float(mm & 0xFFFF0000u));
}

// E8M0 code of a block with max |x| = bm; e = code - 127, eff = g * 2^e.
__device__ __forceinline__ uint32_t q4_scale(float bm, const Q4Global& G, bool& rerr, int& e, float& eff) {
    // s = RN(bm / 448): bm is a bf16 value, so the 3-op division is exact
    // (r = RN(1/448) = 0x1.24924ap-9) while the quotient stays normal
    const float s = bm >= 0x1p-100f ? div1(bm, -kE4M3Max, 0x1.24924ap-9f) : __fdiv_rn(bm, kE4M3Max);
    uint32_t code = 127;
    e = 0;
    if (s > 0.f) {
        const uint32_t sb = __float_as_uint(s);
        if (G.g_normal && sb >= 0x00800000u)
            e = ((int)(sb - G.gbits) + 0x7FFFFF) >> 23;
        else
            e = ceil_log2_ratio(s, G.g);
        if (e < -127) { rerr = true; e = -127; }
        if (e > 127) { rerr = true; e = 127; }
        code = (uint32_t)(e + 127);
    }
    eff = __fmul_rn(G.g, e8m0_to_f32(code));
    return code;
}

// Encode NP pairs of negated values at scale eff -> NP/2 code words (4 codes each, element order).
// General path (a warp with any block outside the fast path's range lands here):
// for any positive finite eff (normal or subnormal f32) write eff = m 2^E, m in
// [1, 2) its significand; then x / eff = (x 2^-E) / m EXACTLY (power-of-two
// scaling) and x 2^-E keeps x's bf16 significand while it stays normal, so the
// 3-op division by m with r = RN(1/m) is again IEEE div.rn.f32 (the proof covers
// every bf16 dividend significand and every f32 divisor significand; all
// magnitudes are now O(1): |x 2^-E| <= 896, no intermediate underflows while the
// quotient is >= 2^-103).  x 2^-E is applied as two exact power-of-two factors
// 2^a 2^b (a, b in [-75, 75]); a product that underflows means a quotient far
// below E4M3's 2^-10 rounding threshold: code +-0 either way, sign kept.  This
// replaced per-element IEEE division, which made late-training gradient tensors
// (tiny block maxima, eff < 2^-60) up to 8x slower to quantize.
template <int NP>
__device__ __forceinline__ void q4_encode(const float (&lo)[NP], const float (&hi)[NP], int e, float eff,
                                          const Q4Global& G, uint32_t (&out)[NP / 2]) {
    const uint32_t eb = __float_as_uint(eff);
    if (eb - 1u < 0x7F7FFFFFu) {                       // 0 < eff < inf
        int E;
        uint32_t mb;
        if (eb >= 0x00800000u) {
            E = (int)(eb >> 23) - 127;
            mb = eb & 0x7FFFFFu;
        } else {                                       // subnormal eff: normalise the significand
            const int lz = __clz(eb) - 8;
            E = -126 - lz;
            mb = (eb << lz) & 0x7FFFFFu;
        }
        const float m = __uint_as_float(mb | 0x3F800000u);
        const float r = __frcp_rn(m);
        const int a = (-E) / 2, bexp = -E - a;         // 2^-E = 2^a 2^b, |a|, |b| <= 75
        const float fa = __uint_as_float((uint32_t)(a + 127) << 23), fb = __uint_as_float((uint32_t)(bexp + 127) << 23);
        const uint64_t nr2 = pk(-r, -r), b2 = pk(m, m), sa = pk(fa, fa), sb = pk(fb, fb);
#pragma unroll
        for (int q = 0; q < NP / 2; ++q) {
            float a0, a1, b0, b1;
            upk(div2n(fmul2(fmul2(pk(lo[2 * q], hi[2 * q]), sa), sb), b2, nr2), a0, a1);
            upk(div2n(fmul2(fmul2(pk(lo[2 * q + 1], hi[2 * q + 1]), sa), sb), b2, nr2), b0, b1);
            out[q] = e4m3x4(a0, a1, b0, b1);
        }
    } else {
#pragma unroll
        for (int q = 0; q < NP / 2; ++q)
            out[q] = e4m3x4(__fdiv_rn(-lo[2 * q], eff), __fdiv_rn(-hi[2 * q], eff), __fdiv_rn(-lo[2 * q + 1], eff),
                            __fdiv_rn(-hi[2 * q + 1], eff));
    }
}

// One 32-element block (16 packed bf16 pairs): unpack, max, E8M0 code, codes.
// Fast path (every block of real data): branch-free scale math —
//   e = ceil(log2(s/g)) = (bits(s) - bits(g) + 0x7FFFFF) >> 23,
//   eff = g 2^e and r = RN(1/g) 2^-e as integer exponent adds (one IMAD each) —
// taken when the whole warp's blocks satisfy bm in {0} u [2^-100, inf) and
// eff = g 2^e in [2^-60, 2^60) (then every value above is exact and equal to
// the general path: see the header).  Otherwise the warp runs q4_scale +
// q4_encode, the general path (one vote per block, no per-thread divergence).
template <int NP>
__device__ __forceinline__ uint32_t q4_block(const uint32_t (&w)[NP], const Q4Global& G, bool& rerr,
                                             uint32_t (&out)[NP / 2]) {
    float lo[NP], hi[NP];
    const float bm = q4_unpack(w, lo, hi);
    const float s = div1(bm, -kE4M3Max, 0x1.24924ap-9f);
    int e = ((int)(__float_as_uint(s) - G.gbits) + 0x7FFFFF) >> 23;
    e = bm > 0.f ? e : 0;
    const bool tiny = (__float_as_uint(bm) - 1u) < (0x0D800000u - 1u);          // 0 < bm < 2^-100
    const bool slow = !G.fast || tiny || (uint32_t)(e - G.emin) > G.erange;
    if (__any_sync(0xFFFFFFFFu, slow)) {
        int e2;
        float eff2;
        const uint32_t code = q4_scale(bm, G, rerr, e2, eff2);
        q4_encode(lo, hi, e2, eff2, G, out);
        return code;
    }
    const float eff = __uint_as_float(G.gbits + (uint32_t)e * 0x00800000u);
    const float r = __uint_as_float(__float_as_uint(G.rg) - (uint32_t)e * 0x00800000u);
    const uint64_t nr2 = pk(-r, -r), b2 = pk(eff, eff);
#pragma unroll
    for (int q = 0; q < NP / 2; ++q) {
        float a0, a1, b0, b1;
        upk(div2n(pk(lo[2 * q], hi[2 * q]), b2, nr2), a0, a1);
        upk(div2n(pk(lo[2 * q + 1], hi[2 * q + 1]), b2, nr2), b0, b1);
        out[q] = e4m3x4(a0, a1, b0, b1);
    }
    return (uint32_t)(e + 127);
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <bool ROW, bool COL, bool MICRO, bool LDSM>
__global__ void __launch_bounds__(Q4_THREADS, 2)
    quant_mx2_v4_kernel(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_codes,
                        const __grid_constant__ CUtensorMap tm_codes_t, int rows, int cols, float* amax_io,
                        int amax_given, uint8_t* __restrict__ sf, uint8_t* __restrict__ micro,
                        uint8_t* __restrict__ sf_t, uint8_t* __restrict__ micro_t, float* g_out, uint32_t* ws,
                        uint32_t* flags, int rev, int dyn, int stagger) {
    extern __shared__ uint8_t q4_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(q4_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* slots = base;                                  // Q4_S x 32 KB
    uint8_t* sfst = base + Q4_S * Q4_IN;                    // 2 x (512 row + 512 col)
    uint64_t* full = reinterpret_cast<uint64_t*>(sfst + 2048);
    __shared__ uint32_t red[Q4_THREADS / 32];
    __shared__ float s_amax;
    __shared__ int slot_tile[Q4_S];

    const int tid = threadIdx.x;
#ifdef Q4_TIMELINE
    unsigned long long tl_t0, tl_t1 = 0, tl_c0;
    int tl_tiles = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_t0));
    tl_c0 = clock64();
#endif
    const int ctiles = cols / Q4_T;
    const int ntiles = ctiles * (rows / Q4_T);
    const int G = gridDim.x, b = blockIdx.x;
    const int n = ntiles > b ? (ntiles - b + G - 1) / G : 0;   // tiles of this CTA: b + j*G
    const int kch_row = cols / 128, kch_t = rows / 128;

    if (tid == 0) {
        prefetch_tmap(&tm_x);
        if (ROW) prefetch_tmap(&tm_codes);
        if (COL) prefetch_tmap(&tm_codes_t);
        for (int s = 0; s < Q4_S; ++s) mbar_init(&full[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto load = [&](int j) {   // tile j of this CTA into slot j % Q4_S (one thread)
        const int tile = b + j * G, s = j % Q4_S;
        const int r0 = (tile / ctiles) * Q4_T, c0 = (tile % ctiles) * Q4_T;
        mbar_arrive_expect_tx(&full[s], Q4_IN);
        tma_load_2d(slots + s * Q4_IN, &tm_x, &full[s], c0, r0);
        tma_load_2d(slots + s * Q4_IN + 16384, &tm_x, &full[s], c0 + 64, r0);
    };
    const bool desc = !amax_given || rev;
    // Producer mode, dynamic schedule (dyn): CTAs take tiles from a global counter in
    // the workspace (atomicAdd by the loading thread, tile index handed to the
    // consumers through slot_tile[] before the barrier arrive), so the CTAs finish
    // together — a static round-robin left a ~25 % tail of idle SMs (per-CTA exit
    // times 80..107 us on a 107 us launch, -DQ4_TIMELINE).  Ordinal k is tile k
    // (ascending) or ntiles-1-k (desc: the producer's last rows are L2-hot).
    // The last CTA to finish resets the counter: no memset, graph-capturable.
    // Hybrid: the first P positions of every CTA are static (ordinal p*G + b: no
    // atomic in the pipeline ramp), the rest come from the counter (ordinal
    // P*G + c), about the last quarter of the tensor — the part where a static
    // schedule's imbalance shows.  The counter is fetched one load ahead
    // (c_next), so the atomic's round trip overlaps a tile instead of delaying
    // the next TMA issue.
    const int P_static = max(Q4_S, (ntiles * 3 / 4) / G);
    int c_next = (dyn && tid == 0) ? (int)atomicAdd(&ws[WS_TILE], 1u) : 0;
    int pos = 0;   // next position to load (loading thread only)
    auto load_dyn = [&](int s) {   // one thread
        int k;
        if (pos < P_static) {
            k = pos * G + b;
        } else {
            k = P_static * G + c_next;
            if (k < ntiles) c_next = (int)atomicAdd(&ws[WS_TILE], 1u);
        }
        ++pos;
        const int tile = k < ntiles ? (desc ? ntiles - 1 - k : k) : -1;
        slot_tile[s] = tile;
        if (tile < 0) {
            mbar_arrive(&full[s]);
            return;
        }
        const int r0 = (tile / ctiles) * Q4_T, c0 = (tile % ctiles) * Q4_T;
        mbar_arrive_expect_tx(&full[s], Q4_IN);
        tma_load_2d(slots + s * Q4_IN, &tm_x, &full[s], c0, r0);
        tma_load_2d(slots + s * Q4_IN + 16384, &tm_x, &full[s], c0 + 64, r0);
    };
    uint32_t par = 0;   // bit s: parity of the next completion of slot s
    auto wait_slot = [&](int s) {
        mbar_wait(&full[s], (par >> s) & 1u);
        par ^= 1u << s;
    };

    // ------------------------------------------------------------ phase A: amax
    // Phase B walks DESCENDING when phase A ran (its last tiles are resident /
    // L2-hot) and, with rev, also in producer mode: the producer kernel that
    // just wrote x finished with its bottom rows, which are the ones still in L2.
    if (!amax_given) {
        if (tid == 0)
            for (int j = 0; j < min(n, Q4_S); ++j) load(j);
        uint32_t m = 0;   // max of (bf16 bits & 0x7FFF) in both halves
        for (int j = 0; j < n; ++j) {
            const int s = j % Q4_S;
            wait_slot(s);
            const uint32_t T = smem_u32(slots + s * Q4_IN) + tid * 16;
#pragma unroll
            for (int q = 0; q < Q4_IN / 16 / Q4_THREADS; ++q) {
                const uint4 u = lds128(T + q * Q4_THREADS * 16);
                m = __vmaxu2(m, u.x & 0x7FFF7FFFu);
                m = __vmaxu2(m, u.y & 0x7FFF7FFFu);
                m = __vmaxu2(m, u.z & 0x7FFF7FFFu);
                m = __vmaxu2(m, u.w & 0x7FFF7FFFu);
            }
            if (j + Q4_S < n) {
                __syncthreads();               // everyone is done with slot s
                if (tid == 0) load(j + Q4_S);
            }
        }
        m = max(m & 0xFFFFu, m >> 16);
        m = __reduce_max_sync(0xFFFFFFFFu, m);
        if ((tid & 31) == 0) red[tid >> 5] = m;
        __syncthreads();
        if (tid == 0) {
            uint32_t r = 0;
            for (int i = 0; i < Q4_THREADS / 32; ++i) r = max(r, red[i]);
            // grid barrier: arrive with this CTA's max, wait for the release
            volatile uint32_t* vws = ws;
            const uint32_t gen = vws[WS_GEN];
            atomicMax(&ws[WS_AMAX0 + (gen & 1u)], r);
            __threadfence();
            const uint32_t old = atomicAdd(&ws[WS_ARRIVE], 1u);
            if (old == (uint32_t)G - 1) {
                ws[WS_ARRIVE] = 0;
                ws[WS_AMAX0 + ((gen + 1u) & 1u)] = 0;    // the next launch's slot
                __threadfence();
                atomicAdd(&ws[WS_GEN], 1u);
            } else {
                uint32_t spins = 0;
                while (ld_acquire_gpu(&ws[WS_GEN]) == gen) {
                    __nanosleep(64);
                    if (++spins > (1u << 26)) __trap();
                }
            }
            __threadfence();
            const uint32_t a16 = vws[WS_AMAX0 + (gen & 1u)];
            if (a16 >= 0x7F80u) {
                if (b == 0) atomicOr(flags, MOSS_FLAG_NONFINITE);
            }
            s_amax = __uint_as_float(a16 << 16);
            if (b == 0) {
                if (amax_io) *amax_io = s_amax;
            }
        }
        __syncthreads();
    } else {
        if (tid == 0) {
            // the tile loads go out before the amax read-back (whose round trip would
            // otherwise delay them); with `stagger` only the first tile of every CTA is
            // requested now and the other two once it has arrived, so the first tiles
            // of all CTAs are not queued behind everybody's second and third
            const int first = stagger ? 1 : Q4_S;
            if (dyn)
                for (int s = 0; s < first; ++s) load_dyn(s);
            else
                for (int j = 0; j < min(n, first); ++j) load(desc ? n - 1 - j : j);
            s_amax = *amax_io;
            if ((__float_as_uint(s_amax) & 0x7F800000u) == 0x7F800000u && b == 0) atomicOr(flags, MOSS_FLAG_NONFINITE);
        }
        __syncthreads();
    }
    const Q4Global Gs = q4_global(s_amax);
    if (g_out && b == 0 && tid == 0) *g_out = Gs.g;

    // ------------------------------------------------------------ phase B: quantize
    // row pass: thread (rr, kb0) owns blocks (rr, kb0) and (rr, kb0 + 2);
    // col pass: thread (rb, cp) owns the 32-row blocks rb of columns 2cp, 2cp+1.
    // (A 512-thread variant with half-blocks per thread measured 25 % slower:
    // the kernel is latency-bound at 16 warps/SM and the split adds per-block work.)
    // All smem offsets are hoisted out of the tile loop: with the SWIZZLE_128B
    // layouts the per-access offset is a per-thread base XOR a compile-time
    // chunk index (the base has zero bits 4-6).
    bool rerr = false;
    const int rr = tid & 127, kb0 = tid >> 7;
    const int rb = tid >> 6, cp = tid & 63;
    // row-pass loads: block kb0 + 2h, 16 B chunk q: rbase ^ (q << 4) + h * 16384
    const uint32_t rbase = (uint32_t)(rr * 128 + ((((kb0 * 4) ^ (rr & 7)) & 7) << 4));
    // row-pass stores: code bytes (kb0 + 2h)*32 + 16j: obase ^ ((4h + j) << 4)
    const uint32_t obase = (uint32_t)(rr * 128 + ((((kb0 * 2) ^ (rr & 7)) & 7) << 4));
    const int sfo_row = ((rr & 31) << 4) + ((rr >> 5) << 2) + kb0;        // + 2h
    uint32_t cbase[8];   // col-pass loads: row rb*32 + i, column 2cp -> cbase[i & 7] + i*128
    uint32_t cob[2];     // col-pass stores: output row c, bytes cb*32 + 16j: cob[h] ^ (j << 4)
    int sfo_col[2], ccol[2], cblk[2];
    if (!LDSM) {
        const int c = 2 * cp;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            cbase[k] = (uint32_t)((c >> 6) * 16384 + rb * 32 * 128 + ((((c >> 3) & 7) ^ k) << 4) + ((c & 7) << 1));
#pragma unroll
        for (int h = 0; h < 2; ++h) { ccol[h] = 2 * cp + h; cblk[h] = rb; }
    } else {
        // ldmatrix.trans column pass: the thread owns the column blocks u = 2 warp + h,
        // each = column 8 m + l/4 (m = 2 (l%4) + (u&1) + 8 ((u>>1)&1), one of the 16
        // 8-column groups) x rows 32 b .. 32 b + 31 (b = ((u>>2) + l%4) & 3); its 16 pair
        // words (rows 2p, 2p+1) arrive from 4 LDSM.x4.trans, pair p = 4k + i from
        // matrix i of load k, whose row j is addressed by lane 8i + j as row
        // 32 b' + 8k + 2i + (j&1) of group m' (b', m' those of quad j>>1).  Conflict-free:
        // a matrix's 8 rows sit in 16-B chunks (m'&7) ^ (2i + (j&1)), all distinct; the
        // code stores of a quad land in distinct chunks (2b) ^ (c&7).
        const int lane = tid & 31, warp = tid >> 5;
        const int ai = lane >> 3, aq = (lane >> 1) & 3, as = lane & 1;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int u = 2 * warp + h;
            const int ma = 2 * aq + (u & 1) + 8 * ((u >> 1) & 1), ba = ((u >> 2) + aq) & 3;
            const int ra = 32 * ba + 2 * ai + as;
            cbase[h] = (uint32_t)((ma >> 3) * 16384 + ra * 128 + (((ma & 7) ^ (ra & 7)) << 4));
            const int qd = lane & 3;
            const int mo = 2 * qd + (u & 1) + 8 * ((u >> 1) & 1);
            ccol[h] = 8 * mo + (lane >> 2);
            cblk[h] = ((u >> 2) + qd) & 3;
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int c = ccol[h];
        cob[h] = (uint32_t)(c * 128 + ((((cblk[h] * 2) ^ (c & 7)) & 7) << 4));
        sfo_col[h] = 512 + ((c & 31) << 4) + ((c >> 5) << 2) + cblk[h];
    }
    for (int p = 0; dyn || p < n; ++p) {
        const int j = desc ? n - 1 - p : p;
        const int s = dyn ? p % Q4_S : j % Q4_S;
        if (amax_given || p >= Q4_S) wait_slot(s);    // phase A's resident tiles were waited there
        if (amax_given && stagger && p == 0 && tid == 0) {   // the deferred initial loads
            if (dyn) {
                for (int s2 = 1; s2 < Q4_S; ++s2) load_dyn(s2);
            } else {
                for (int j2 = 1; j2 < min(n, Q4_S); ++j2) load(desc ? n - 1 - j2 : j2);
            }
        }
        const int tile = dyn ? slot_tile[s] : b + j * G;
        if (tile < 0) break;                           // dyn: the counter ran out (CTA-uniform)
#ifdef Q4_TIMELINE
        tl_tiles = p + 1;
#endif
#ifdef Q4_TIMELINE
        if (p == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_t1));
#endif
        uint8_t* Tg = slots + s * Q4_IN;               // generic: for the TMA store
        const uint32_t T = smem_u32(Tg);
        uint8_t* sfsg = sfst + (p & 1) * 1024;
        const uint32_t sfs = smem_u32(sfsg);
        const int r0 = (tile / ctiles) * Q4_T, c0 = (tile % ctiles) * Q4_T;

        uint32_t ucol[32];
        if (COL) {
            if (LDSM) {
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        ldsm4t(T + cbase[h] + k * 1024, ucol[16 * h + 4 * k], ucol[16 * h + 4 * k + 1],
                               ucol[16 * h + 4 * k + 2], ucol[16 * h + 4 * k + 3]);
            } else {
#pragma unroll
                for (int i = 0; i < 32; ++i) ucol[i] = lds32(T + cbase[i & 7] + i * 128);
            }
        }
        uint32_t rcodes[2][8];
        if (ROW) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                uint32_t w[16];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint4 u = lds128(T + h * 16384 + (rbase ^ (uint32_t)(q << 4)));
                    w[4 * q] = u.x; w[4 * q + 1] = u.y; w[4 * q + 2] = u.z; w[4 * q + 3] = u.w;
                }
                const uint32_t code = q4_block(w, Gs, rerr, rcodes[h]);
                sts8(sfs + sfo_row + 2 * h, code);
                if (MICRO && micro) micro[(int64_t)(r0 + rr) * (cols >> 5) + (c0 >> 5) + kb0 + 2 * h] = (uint8_t)code;
            }
        }
        __syncthreads();                           // the whole tile is in registers: reuse the slot for codes
        if (ROW) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                sts128(T + (obase ^ (uint32_t)((4 * h) << 4)), rcodes[h][0], rcodes[h][1], rcodes[h][2], rcodes[h][3]);
                sts128(T + (obase ^ (uint32_t)((4 * h + 1) << 4)), rcodes[h][4], rcodes[h][5], rcodes[h][6],
                       rcodes[h][7]);
            }
        }
        if (COL) {
            const uint32_t Tc = T + 16384;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                // column ccol[h]: rows 2i, 2i+1 of the block packed as one pair word
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 16; ++i)
                    w[i] = LDSM ? ucol[16 * h + i]
                                : (h ? __byte_perm(ucol[2 * i], ucol[2 * i + 1], 0x7632)
                                     : __byte_perm(ucol[2 * i], ucol[2 * i + 1], 0x5410));
                uint32_t cc[8];
                const uint32_t code = q4_block(w, Gs, rerr, cc);
                sts128(Tc + cob[h], cc[0], cc[1], cc[2], cc[3]);
                sts128(Tc + (cob[h] ^ 16u), cc[4], cc[5], cc[6], cc[7]);
                sts8(sfs + sfo_col[h], code);
                if (MICRO && micro_t)
                    micro_t[(int64_t)(c0 + ccol[h]) * (rows >> 5) + (r0 >> 5) + cblk[h]] = (uint8_t)code;
            }
        }
        fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            if (ROW) {
                tma_store_2d(&tm_codes, Tg, c0, r0);
                if (sf) bulk_store(sf + ((int64_t)(r0 >> 7) * kch_row + (c0 >> 7)) * 512, sfsg, 512);
            }
            if (COL) {
                tma_store_2d(&tm_codes_t, Tg + 16384, r0, c0);
                if (sf_t) bulk_store(sf_t + ((int64_t)(c0 >> 7) * kch_t + (r0 >> 7)) * 512, sfsg + 512, 512);
            }
            bulk_commit();
            // the store of position p-1 has read its slot and SF staging -> refill the slot with p+2
            if (p >= 1) {
                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                if (dyn)
                    load_dyn((p + 2) % Q4_S);
                else if (p + 2 < n)
                    load(desc ? n - 1 - (p + 2) : p + 2);
            }
        }
    }
    if (tid == 0) {
        bulk_wait0();
        if (dyn) {
            // every fetch of this CTA precedes its arrival here; the last CTA resets
            __threadfence();
            if (atomicAdd(&ws[WS_DONE], 1u) == (uint32_t)G - 1) {
                ws[WS_TILE] = 0;
                ws[WS_DONE] = 0;
            }
        }
    }
    if (__any_sync(0xFFFFFFFFu, rerr) && (tid & 31) == 0) atomicOr(flags, MOSS_FLAG_E8M0_RANGE);
#ifdef Q4_TIMELINE
    if (tid == 0 && b < 1024) {
        unsigned long long t2;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        unsigned long long* o = q4_tl + b * 8;
        o[0] = tl_t0; o[1] = tl_t1; o[2] = t2; o[3] = clock64() - tl_c0; o[4] = smid; o[5] = tl_tiles;
        o[6] = (unsigned long long)rows * cols; o[7] = G;
    }
#endif
}

// returns false when the shape/dtype is not covered (caller falls back)
// MOSS_Q4_REV=0 walks producer-mode tiles in ascending order (A/B on the box)
static int q4_rev() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_Q4_REV");
        v = e ? (e[0] != '0') : 1;
    }
    return v;
}

// MOSS_Q4_STAGGER=0: producer mode requests all three initial tiles at once (A/B; read per launch)
static int q4_stagger() {
    const char* e = getenv("MOSS_Q4_STAGGER");
    return e ? (e[0] != '0') : 1;
}

// MOSS_Q4_DYN=0: static round-robin tiles in producer mode; =2: the dynamic tail at
// every size (tests, sanitizers).  Read at every launch: A/B inside one process,
// e.g. two graphs captured under each setting.
static int q4_dyn() {
    const char* e = getenv("MOSS_Q4_DYN");
    return e ? (e[0] == '2' ? 2 : e[0] != '0') : 1;
}

// MOSS_Q4_LDSM=0 selects the LDS.32 + PRMT column loads (A/B on the box)
static int q4_ldsm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("MOSS_Q4_LDSM");
        v = e ? (e[0] != '0') : 1;
    }
    return v;
}

bool launch_quant_v4(const void* x, int64_t rows, int64_t cols, float* amax, int amax_given, uint8_t* codes,
                     uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                     uint32_t* ws, uint32_t* flags, cudaStream_t st, int* status) {
    *status = MOSS_OK;
    if (rows % Q4_T || cols % Q4_T || rows > INT32_MAX || cols > INT32_MAX) return false;
    const bool row = codes != nullptr;
    const bool col = codes_t != nullptr;
    if ((!row && (sf || micro)) || (!col && (sf_t || micro_t)) || (!row && !col)) return false;
    if (!amax_given && !ws) return false;
    CUtensorMap mx, mc, mct;
    if (!make_tmap_2d(&mx, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, rows, cols, 64, Q4_T, CU_TENSOR_MAP_SWIZZLE_128B))
        return false;
    mc = mx;
    mct = mx;
    if (row && !make_tmap_2d(&mc, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, codes, rows, cols, Q4_T, Q4_T,
                             CU_TENSOR_MAP_SWIZZLE_128B))
        return false;
    if (col && !make_tmap_2d(&mct, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, codes_t, cols, rows, Q4_T, Q4_T,
                             CU_TENSOR_MAP_SWIZZLE_128B))
        return false;
    const bool mic = micro || micro_t;
    using KT = decltype(&quant_mx2_v4_kernel<true, true, true, true>);
    static const KT kernels[12] = {
        quant_mx2_v4_kernel<true, true, false, false>, quant_mx2_v4_kernel<false, true, false, false>,
        quant_mx2_v4_kernel<true, false, false, false>, quant_mx2_v4_kernel<true, true, true, false>,
        quant_mx2_v4_kernel<false, true, true, false>, quant_mx2_v4_kernel<true, false, true, false>,
        quant_mx2_v4_kernel<true, true, false, true>, quant_mx2_v4_kernel<false, true, false, true>,
        quant_mx2_v4_kernel<true, false, false, true>, quant_mx2_v4_kernel<true, true, true, true>,
        quant_mx2_v4_kernel<false, true, true, true>, quant_mx2_v4_kernel<true, false, true, true>};
    const int ki = (row && col ? 0 : (col ? 1 : 2)) + (mic ? 3 : 0) + (q4_ldsm() ? 6 : 0);

    const KT kern = kernels[ki];
    static int occ_dev[kMaxDevices][12] = {};
    int* occ = occ_dev[current_device()];
    if (!occ[ki]) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Q4_SMEM) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[ki], kern, Q4_THREADS, Q4_SMEM) != cudaSuccess ||
            occ[ki] < 1) {
            occ[ki] = 0;
            *status = MOSS_ERR_CUDA;
            return true;
        }
    }
    const int64_t ntiles = (rows / Q4_T) * (cols / Q4_T);
    const int grid = (int)std::min<int64_t>(ntiles, (int64_t)sm_count() * occ[ki]);
    // dynamic tail only for big tensors (>= 8 tiles per CTA): standalone 8192 x {11008, 12288,
    // 22016} +6-9 %; at <= 7 tiles per CTA the counter's atomics cost more than the tail
    // (4096^2: 22.5 vs 20.5 us); in the layer step's graph the two schedules measured equal
    const int dm = q4_dyn();
    const int dyn = amax_given && ws && dm && (dm == 2 || ntiles >= 8 * (int64_t)grid);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(Q4_THREADS);
    cfg.dynamicSmemBytes = Q4_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    // the amax phase ends in a grid-wide barrier: all CTAs must be co-resident
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = amax_given ? 0 : 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, mx, mc, mct, (int)rows, (int)cols, amax, amax_given, sf,
                                             micro, sf_t, micro_t, g_out, ws, flags, q4_rev(), dyn, q4_stagger());
    *status = e == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
    return true;
}

}  // namespace moss

#ifdef Q4_TIMELINE
extern "C" int moss_q4_timeline(void* host_dst) {
    return cudaMemcpyFromSymbol(host_dst, moss::q4_tl, sizeof(moss::q4_tl)) == cudaSuccess ? 0 : 5;
}
#endif
