/* CPU ORACLE — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * C restatement of the reference codec and two-level quantizer
 * (/root/reference/pkg/src/mossq/fp8.py:131-183, 194-223 and
 *  quantize.py:92-98, 127-173), used by tests/ for parity at BASELINE sizes
 * (numpy needs seconds per 4096^2 tensor; this needs milliseconds) and for
 * the exhaustive 2^32 codec sweep.  It is itself pinned against the numpy
 * restatement and the reference's golden vectors in tests/test_oracle.py.
 *
 * Build: oracle/Makefile -> oracle/_build/libmoss_oracle.so (gcc -O2, no
 * fast-math: every f32 division below must be IEEE round-to-nearest).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

static inline uint32_t f2u(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static inline float u2f(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* fp8.py:131-183 for E4M3 (bias 7, 3 mantissa bits, max 448 = code 0x7E):
 * round-to-nearest-even on the target significand, saturate to max finite,
 * f32 subnormals and zeros -> signed zero.  Non-finite input is the caller's
 * problem (the reference raises before encoding). */
uint8_t moss_oracle_e4m3(float x) {
    uint32_t b = f2u(x);
    uint8_t sign = (uint8_t)((b >> 24) & 0x80u);
    int fexp = (int)((b >> 23) & 0xFFu);
    if (fexp == 0) return sign;                      /* zero or f32 subnormal */
    uint64_t sig = (uint64_t)((b & 0x7FFFFFu) | 0x800000u);
    int tgt = fexp - 127 + 7;                        /* biased E4M3 exponent */
    int shift = 20 + (tgt < 1 ? 1 - tgt : 0);
    if (shift > 60) shift = 60;
    uint64_t q = sig >> shift;
    uint64_t rem = sig & ((1ull << shift) - 1ull);
    uint64_t half = 1ull << (shift - 1);
    if (rem > half || (rem == half && (q & 1ull))) q += 1;
    if (q == 16) { q >>= 1; tgt += 1; }              /* carry into next binade */
    int e_out, m_out;
    if (q >= 8) { e_out = tgt < 1 ? 1 : tgt; m_out = (int)q - 8; }
    else        { e_out = 0;                 m_out = (int)q;     }
    if (e_out > 15 || (e_out == 15 && m_out > 6)) { e_out = 15; m_out = 6; }
    return (uint8_t)(sign | (e_out << 3) | m_out);
}

/* Encode n floats; returns the number of non-finite inputs seen. */
int64_t moss_oracle_e4m3_array(const float* x, uint8_t* out, int64_t n) {
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(x[i])) { ++bad; out[i] = 0x7F; continue; }
        out[i] = moss_oracle_e4m3(x[i]);
    }
    return bad;
}

/* Exhaustive sweep helper: encode every f32 bit pattern in [lo, hi) and
 * compare against a device-produced table; returns mismatches. */
int64_t moss_oracle_e4m3_sweep_compare(uint32_t lo, uint64_t hi, const uint8_t* dev) {
    int64_t bad = 0;
    for (uint64_t u = lo; u < hi; ++u) {
        float f = u2f((uint32_t)u);
        uint8_t want = isfinite(f) ? moss_oracle_e4m3(f) : dev[u - lo];
        if (dev[u - lo] != want) ++bad;
    }
    return bad;
}

/* ceil_pow2 exponent of s/g computed exactly from the f32 bit patterns
 * (equivalent to fp8.py:205-208 frexp on the f64 quotient).  s, g > 0. */
static int ceil_log2_ratio(float s, float g) {
    int es, eg;
    float ms = frexpf(s, &es);   /* s = ms * 2^es, ms in [0.5, 1) exact */
    float mg = frexpf(g, &eg);
    int e = es - eg;             /* ratio in (2^(e-1), 2^(e+1)) */
    if (ms > mg) return e + 1;   /* ratio in (2^e, 2^(e+1)) -> e+1 */
    return e;                                         /* ms <= mg: ratio in (2^(e-1), 2^e] */
}

/* The per-block part of quantize.py:144-173 for rows x cols at a given
 * global scale g (row ranges of one tensor can be done independently). */
int moss_oracle_quant_two_level_rows(const float* x, int64_t rows, int64_t cols, float g,
                                     uint8_t* codes, uint8_t* micro) {
    const int64_t nb = cols / 32;
    int status = 0;
    for (int64_t r = 0; r < rows; ++r) {
        for (int64_t b = 0; b < nb; ++b) {
            const float* blk = x + r * cols + b * 32;
            float bmax = 0.f;
            for (int j = 0; j < 32; ++j) { float a = fabsf(blk[j]); if (a > bmax) bmax = a; }
            float s = bmax / 448.0f;
            int e = 0;
            uint8_t mc = 127;
            if (s > 0.f) {
                e = ceil_log2_ratio(s, g);
                if (e < -127 || e > 127) { status = 2; e = e < -127 ? -127 : 127; }
                mc = (uint8_t)(e + 127);
            }
            micro[r * nb + b] = mc;
            float eff = g * ldexpf(1.0f, (int)mc - 127);
            for (int j = 0; j < 32; ++j)
                codes[r * cols + b * 32 + j] = moss_oracle_e4m3(blk[j] / eff);
        }
    }
    return status;
}

/* quantize.py:127-173, rows x cols f32 row-major, blocks of 32 along cols.
 * amax over the whole tensor is computed here.  Outputs: codes[rows*cols],
 * micro[rows*cols/32] (row-major), *g_out.  Returns 0, or 1 for non-finite
 * input, 2 for an E8M0 exponent below -127 (the reference raises). */
int moss_oracle_quant_two_level(const float* x, int64_t rows, int64_t cols,
                                uint8_t* codes, uint8_t* micro, float* g_out) {
    float amax = 0.f;
    for (int64_t i = 0; i < rows * cols; ++i) {
        if (!isfinite(x[i])) return 1;
        float a = fabsf(x[i]);
        if (a > amax) amax = a;
    }
    float g = amax > 0.f ? amax / 448.0f : 1.0f;      /* == max_i f32(bmax_i/448) */
    if (g == 0.f) g = 1.0f;
    *g_out = g;
    return moss_oracle_quant_two_level_rows(x, rows, cols, g, codes, micro);
}

/* Weight copy at a given scale, train.py:113-118: codes = e4m3(f32(w)/f32(s)). */
int64_t moss_oracle_encode_scaled(const float* w, int64_t n, float scale, uint8_t* codes) {
    int64_t sat = 0;
    float lim = scale * 448.0f;
    for (int64_t i = 0; i < n; ++i) {
        if (fabsf(w[i]) > lim) ++sat;
        codes[i] = moss_oracle_e4m3(w[i] / scale);
    }
    return sat;
}
