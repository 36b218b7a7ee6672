/* Exhaustive check of the quantizer's 3-op division (csrc/quant_v4.cu):
 *   q0 = RN(x * r), rem = fma(b, q0, -x), q = fma(-r, rem, q0),  r = RN(1/b)
 * equals the IEEE quotient RN(x / b) for EVERY f32 divisor significand
 * b in [1, 2) (2^23 values) and EVERY bf16 dividend significand x in
 * [1, 4) (256 values: two binades, so quotients on both sides of 1 are
 * covered).  Power-of-two scaling of x and b is exact while all values stay
 * normal, so this covers every normal bf16 / f32 pair.  Also checks the
 * constant RN(1/448) used for s_i = RN(bmax / 448).
 * Prints "mismatches <n>" and exits 0 iff n == 0. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

static float fb(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }
static uint32_t bf(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

int main(void) {
    long bad = 0;
#pragma omp parallel for reduction(+ : bad) schedule(dynamic, 4096)
    for (uint32_t mb = 0; mb < (1u << 23); ++mb) {
        const float b = fb(0x3F800000u | mb);
        const float r = 1.0f / b;  /* IEEE RN(1/b) == __frcp_rn */
        for (uint32_t mx = 0; mx < 256; ++mx) {
            const float x = fb((mx < 128 ? 0x3F800000u : 0x40000000u) | ((mx & 127u) << 16));
            const float q0 = x * r;
            const float q = fmaf(-r, fmaf(b, q0, -x), q0);
            if (bf(q) != bf(x / b)) bad++;
            /* the kernel evaluates it on -x with -r: same bits, signed zeros kept */
            const float xn = -x, q0n = xn * -r;
            const float qn = fmaf(-r, fmaf(b, q0n, xn), q0n);
            if (bf(qn) != bf(x / b)) bad++;
        }
    }
    if (bf(1.0f / 448.0f) != 0x3B124925u) bad++;   /* 0x1.24924ap-9 */
    {   /* signed zero: x = -0 must give -0 (E4M3 0x80, quantize.py:171 / fp8.py:148-149) */
        const float xn = 0.0f, r = 1.0f / 1.75f, q0 = xn * -r;
        if (bf(fmaf(-r, fmaf(1.75f, q0, xn), q0)) != 0x80000000u) bad++;
    }
    printf("mismatches %ld\n", bad);
    return bad != 0;
}
