/* moss_b200.h — C ABI of the B200-native MOSS FP8 training hot path.
 *
 * Plain pointers and sizes only: every pointer is a DEVICE pointer unless
 * stated otherwise, every call is stream-ordered on the given cudaStream_t
 * (passed as void*), nothing allocates, frees or synchronises.  The library
 * is loaded with ctypes by paper_2511_05811_b200/_lib.py; INTEGRATION.md shows
 * the binding a maintainer would add to the reference.
 *
 * Each entry point names the reference interface it replaces
 * (paths under /root/reference/pkg/src/mossq/).
 *
 * Status codes mirror the reference's exception classes (errors.py:4-45):
 * host-checkable problems are returned before launch; data-dependent ones
 * (non-finite input, E8M0 exponent < -127) are OR-ed into *flags on the
 * device and raised by the host at the next check.
 */
#ifndef MOSS_B200_H
#define MOSS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum moss_status {
    MOSS_OK = 0,
    MOSS_ERR_SHAPE = 1,     /* InvalidShapeError   */
    MOSS_ERR_VALUE = 2,     /* InvalidValueError   */
    MOSS_ERR_ARGUMENT = 3,  /* InvalidArgumentError */
    MOSS_ERR_E8M0 = 4,      /* E8m0RangeError      */
    MOSS_ERR_CUDA = 5,      /* CUDA runtime failure */
    MOSS_ERR_ALIGN = 6      /* pointer / stride alignment (InvalidArgumentError) */
};

enum moss_dtype { MOSS_F32 = 0, MOSS_BF16 = 1 };

/* device flag bits */
#define MOSS_FLAG_NONFINITE 1u      /* NaN/Inf input: quantize.py:88, fp8.py:139 */
#define MOSS_FLAG_E8M0_RANGE 2u     /* e8m0 exponent < -127: fp8.py:219-222 */
#define MOSS_FLAG_GRAD_NONFINITE 4u /* optim.py:89-90 */
/* Any of these bits set when K3 starts => K3 skips its whole update (no
 * write to w, m, v, codes or scale_out): the reference raises before it
 * mutates anything (quantize.py:88, fp8.py:219-222, optim.py:89-90).  K3
 * with p->step != 0 then also atomicMin()s p->step into flags[1], so a
 * caller that passes step numbers must give K3 a TWO-word flags buffer,
 * flags[1] initialised to 0xFFFFFFFF (= "no step skipped"). */
#define MOSS_FLAG_SKIP_MASK (MOSS_FLAG_NONFINITE | MOSS_FLAG_E8M0_RANGE | MOSS_FLAG_GRAD_NONFINITE)

/* Bytes of the tcgen05 block-scale-factor buffer for a rows x cols operand
 * (one E8M0 byte per 32 columns; 128-row x 4-block chunks of 512 B). */
int64_t moss_sf_bytes(int64_t rows, int64_t cols);

/* K0: amax = max|x| over n elements (f32 bits, written with atomicMax after a
 * stream-ordered memset of *amax to 0).  Non-finite elements set
 * MOSS_FLAG_NONFINITE.  Replaces the max-reductions of quantize.py:95 / 149-151
 * and autoscale.py:58 (jit_scale).  Reads x back to front so that the
 * following quantizer finds the head of x still in L2. */
int moss_amax(const void* x, int dtype, int64_t n, float* amax, uint32_t* flags, void* stream);

/* K1: two-level MOSS quantization, quant_two_level(x, E4M3, CEIL_POW2, k2=32,
 * k1=None) (quantize.py:127-173), of a rows x cols row-major tensor.
 *   amax         device f32 from moss_amax (g = f32(amax/448), 0 -> 1.0)
 *   codes        [rows, cols] E4M3 codes, blocks of 32 along cols   (nullable)
 *   sf           block-scale layout for the GEMM, moss_sf_bytes(rows, cols) (nullable)
 *   micro        [rows, cols/32] row-major E8M0 codes (the reference layout) (nullable)
 *   codes_t      [cols, rows] codes of quant_two_level(x.T): blocks of 32 along
 *                rows (the wgrad operand), same g                  (nullable)
 *   sf_t, micro_t  scales of codes_t, layouts as above              (nullable)
 *   g_out        device f32 global scale (nullable)
 * cols % 32 == 0; if codes_t/sf_t/micro_t is given also rows % 32 == 0. */
int moss_quant_mx2(const void* x, int dtype, int64_t rows, int64_t cols, const float* amax,
                   uint8_t* codes, uint8_t* sf, uint8_t* micro,
                   uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                   float* g_out, uint32_t* flags, void* stream);

/* K0+K1 in ONE launch (single pass over HBM for tensors that fit in L2 +
 * smem): the same outputs as moss_amax followed by moss_quant_mx2, i.e.
 * quant_two_level (quantize.py:127-173) including the global amax
 * (quantize.py:149-155).  The kernel streams x once to reduce max|x|, meets
 * all CTAs at one grid-wide barrier (cooperative launch), then quantizes the
 * tiles still resident in shared memory / L2 first.
 *   amax         amax_given == 0: OUT, max|x| (f32) of the tensor;
 *                amax_given != 0: IN, max|x| supplied by the producer kernel
 *                (producer-fused amax: the quantizer then reads x once and
 *                skips the reduction and the barrier)
 *   workspace    moss_workspace_bytes() bytes of device memory, zeroed once
 *                by the caller and reused; one stream at a time per workspace
 *                (grid-barrier words of the in-kernel amax; in producer mode the
 *                tile counter of the load-balanced tail; both reset by the
 *                kernel's last CTA, so the words are zero between launches)
 *   other arguments as moss_quant_mx2.
 * bf16 tensors with rows % 128 == 0 and cols % 128 == 0 take the fused
 * kernel; other shapes/dtypes run moss_amax + moss_quant_mx2 internally. */
int moss_quant_mx2_fused(const void* x, int dtype, int64_t rows, int64_t cols, float* amax, int amax_given,
                         uint8_t* codes, uint8_t* sf, uint8_t* micro,
                         uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                         float* g_out, uint32_t* workspace, uint32_t* flags, void* stream);

/* Bytes of the caller-owned workspace of moss_quant_mx2_fused. */
int64_t moss_workspace_bytes(void);

/* Per-tensor encode at a given scale: codes = e4m3(f32(x) / f32(scale))
 * (train.py:113-118 _quantize_weight, quant_per_tensor quantize.py:92-98 when
 * scale = f32(amax/448), rescale_interval autoscale.py:86-96).
 *   scale        device f32 (nullable: then scale_host is used; if also
 *                scale_from_amax != 0, *scale is an amax and the scale is
 *                f32(amax/448), 0 -> 1.0)
 *   codes        [rows, cols] (nullable), codes_t [cols, rows] (nullable)
 *   scale_out    device f32 receiving the scale actually used (nullable)
 *   n_saturated  device u32 counter of |x| > scale*448 (nullable)          */
int moss_encode_scaled(const void* x, int dtype, int64_t rows, int64_t cols, const float* scale,
                       float scale_host, int scale_from_amax, uint8_t* codes, uint8_t* codes_t,
                       float* scale_out, uint32_t* n_saturated, uint32_t* flags, void* stream);

/* K2: block-scaled MXFP8 GEMM on tcgen05 (kind::mxf8f6f4, E8M0 scales in TMEM,
 * FP32 accumulate), the dataflow of gemm_mx_epilogue (gemm.py:115-129):
 *   D[m, n] = (sum_k A[m,k] 2^(SFA[m,k/32]-127) B[n,k] 2^(SFB[n,k/32]-127)) * (*sA) * (*sB)
 * A [M,K] and B [N,K] are K-major E4M3 codes; SFA/SFB in the block-scale
 * layout (SFB == NULL means unit scales: the per-tensor weight side,
 * PAPER.md:103).  D is [M, N] row-major (ldd elements), bf16 or f32;
 * accumulate != 0 adds into D (f32 only).  K % 128 == 0, M, N >= 1.
 * d_amax (nullable): receives max|D| of the stored values as f32 (zeroed by the
 * call; the amax epilogue for the quantizer that consumes D, quantize.py:149-155
 * — not with accumulate, and D contiguous (ldd == N)); flags receives
 * MOSS_FLAG_NONFINITE from the separate amax pass of the 1-CTA fallback.
 * The reference returns (out_features, tokens): call with A = weights,
 * B = activations for that orientation, or A = activations for torch's. */
int moss_gemm_mxf8(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB,
                   const float* sA, const float* sB, void* D, int d_dtype, int64_t ldd,
                   int64_t M, int64_t N, int64_t K, int accumulate, float* d_amax, uint32_t* flags, void* stream);

/* K3 hyper-parameters of one AdamW step (optim.py:52-62, 78-106). */
typedef struct {
    float lr;         /* eta_t */
    float beta1, beta2;
    float eps;
    float weight_decay;
    float bc1, bc2;   /* 1 - beta1^t, 1 - beta2^t for the step being taken */
    int decoupled;    /* 1 = AdamW (decay on the old weight), 0 = L2 into g */
    float grad_scale; /* g is multiplied by this first (DP averaging, grad accumulation); 1 = none */
    uint32_t step;    /* optimizer step number t (>= 1) recorded in flags[1] when the update is skipped; 0 = don't */
} moss_adam_params;

/* Sets `bit` in *flags if any of the n elements of x (f32 or bf16) is NaN/Inf.
 * The optimizer runs it over the gradients K3's gate cannot vouch for (those
 * not produced from flag-checked FP8 operands) BEFORE any K3 launch of the
 * step, so a non-finite gradient skips every update of the step
 * (optim.py:89-90 raises before mutating). */
int moss_check_finite(const void* x, int dtype, int64_t n, uint32_t bit, uint32_t* flags, void* stream);

/* moss_gemm_mxf8 with B given as stored [K, N] row-major (N contiguous) and unit
 * B scales: the dgrad product dX = dY W reads the per-tensor E4M3 weight codes
 * W [out = K, in = N] directly (MN-major tcgen05 operand) — no transposed copy
 * of W is kept (replaces the W^T operand of gemm.py:115-129 in the backward).
 * M % 256, N % 256, K % 128.  d_amax (nullable): max|D| as for moss_gemm_mxf8 — the
 * dgrad output is the next layer's output-gradient, quantized next. */
int moss_gemm_mxf8_bkn(const uint8_t* A, const uint8_t* SFA, const uint8_t* B_kn, const float* sA, const float* sB,
                       void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, float* d_amax,
                       void* stream);

/* K3: fused AdamW + automatic scaling + FP8 weight copy
 * (adamw_step optim.py:78-106, then _quantize_weight train.py:113-118 at the
 * advanced scale s_{t+1} = s_t + eta/448, autoscale.py:71-79).
 * w, m, v   f32 [rows, cols] updated in place; g f32 or bf16.
 * enc_scale f32(s_{t+1}) used for w_fp8 = e4m3(w'/enc_scale) (nullable outputs).
 * w_fp8_t   [cols, rows] transposed codes for dgrad (nullable).
 * w_amax    device f32 max|w'| (nullable; memset by the call) — rescale input.
 * n_saturated  device u32 count of |w'| > enc_scale*448 (nullable).
 * If *flags has any MOSS_FLAG_SKIP_MASK bit set when the kernel starts, nothing
 * is written (see MOSS_FLAG_SKIP_MASK).  Elements whose gradient is non-finite
 * are left untouched and set MOSS_FLAG_GRAD_NONFINITE (a gradient that was not
 * checked by moss_check_finite first: the rest of that launch still updates). */
int moss_adamw_fp8(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                   const moss_adam_params* p, float enc_scale, uint8_t* w_fp8, uint8_t* w_fp8_t,
                   float* w_amax, uint32_t* n_saturated, uint32_t* flags, void* stream);

/* K3 with device-resident hyper-parameters, for CUDA-graph replay: *p_dev
 * and *enc_scale_dev are read by the kernel (the host refreshes them with a
 * stream-ordered H2D copy before each replay).  scale_out (nullable) receives
 * *enc_scale_dev when the update is done — the f32(s_{t+1}) the next forward's
 * GEMMs read as the weight's per-tensor scale. */
int moss_adamw_fp8_dev(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                       const moss_adam_params* p_dev, const float* enc_scale_dev, float* scale_out,
                       uint8_t* w_fp8, uint8_t* w_fp8_t, float* w_amax, uint32_t* n_saturated,
                       uint32_t* flags, void* stream);

/* ---------------------------------------------------------------------------
 * Producer kernels (bf16): the Llama ops that make every FP8 linear's input
 * and output-gradient, each also writing max|output| to *amax (nullable;
 * zeroed by the call) so that moss_quant_mx2_fused runs with amax_given = 1
 * (producer-fused amax).  Not reference functions:
 * the reference's training harness is a 2-layer MLP (train.py:126-204); these
 * implement the decoder the north_star trains.  All tensors row-major.
 *
 * RMSNorm over the last dim d (d % 8 == 0, d <= 8192), T rows:
 *   x' = x + delta (bf16; written to x_out when delta != NULL)
 *   y  = x' * rsqrt(mean(x'^2) + eps) * w   (f32 math, bf16 out), rstd[T] f32 */
int moss_rmsnorm_fwd(const void* x, const void* delta, void* x_out, const float* w, float eps, void* y, float* rstd,
                     float* amax, int64_t T, int64_t d, void* stream);
/*   dx = rstd (dy w - xh mean(dy w xh)) + d_res   (xh = x' rstd; d_res nullable)
 *   dw += sum_t dy xh  (f32, accumulated in a fixed order — deterministic;
 *   dw nullable).  workspace: moss_rmsnorm_bwd_workspace_bytes(T, d) bytes. */
int moss_rmsnorm_bwd(const void* dy, const void* x, const float* w, const float* rstd, const void* d_res, void* dx,
                     float* dw, float* amax, float* workspace, int64_t T, int64_t d, void* stream);
int64_t moss_rmsnorm_bwd_workspace_bytes(int64_t T, int64_t d);
/* SwiGLU on gu = [gate | up] (T x 2f): h = silu(gate) * up (T x f) */
int moss_swiglu_fwd(const void* gu, void* h, float* amax, int64_t T, int64_t f, void* stream);
/* dgu = [dh up silu'(gate) | dh silu(gate)] */
int moss_swiglu_bwd(const void* dh, const void* gu, void* dgu, float* amax, int64_t T, int64_t f, void* stream);
/* RoPE: qkv [B, S, 3, H, hd] -> q, k, v, q/k pairs (2i, 2i+1) rotated by
 * cos/sin [S_max, hd/2] (f32) at position s.  q, k, v memory: [B, H, S, hd]
 * (bshd = 0) or [B, S, H, hd] (bshd = 1; SDPA then returns its output in that
 * layout and the O projection reads it without a transpose copy). */
int moss_rope_fwd(const void* qkv, const float* cosv, const float* sinv, void* q, void* k, void* v, int64_t B,
                  int64_t S, int64_t H, int64_t hd, int bshd, void* stream);
/* Elementwise glue producers (bf16, f32 math), each writing max|out| to *amax:
 * mode 0 sum3:   out [T, d] = x[:, 0:d] + x[:, d:2d] + x[:, 2d:3d]   (x [T, 3d])
 * mode 1 bcast3: out [T, 3d] = [x, x, x]                              (x [T, d])
 * mode 2 add:    out = x + y
 * mode 3 scale:  out = (x [+ y]) * f32(*scale * alpha)                (scale: device f32, e.g. the
 *                incoming loss gradient; alpha: host factor, e.g. 2/n for mean((x + y)^2);
 *                y optional: a fixed offset) */
int moss_glue(int mode, const void* x, const void* y, const float* scale, float alpha, void* out, float* amax,
              int64_t T, int64_t d, void* stream);
/* *acc = scale * sum (x [+ y])^2 (f32) over n bf16 elements (n % 8 == 0; scale = 1/n gives the mean;
 * y optional, same shape: a fixed offset); deterministic (fixed-order reduction through `partials`,
 * MOSS_SUMSQ_PARTIALS floats of caller scratch) */
#define MOSS_SUMSQ_PARTIALS 1024
int moss_sumsq(const void* x, const void* y, int64_t n, float scale, float* acc, float* partials, void* stream);
/* Cross entropy of bf16 logits [T, V] (V % 8 == 0) against int64 targets:
 * fwd  lse[t] = logsumexp(x[t, :]) (f32, one read of the row), loss[t] = lse[t] - x[t, y_t]
 * bwd  dlogits = (softmax(x) - onehot(y)) * (*scale), bf16; scale a device f32 (dL/dmean / T) */
int moss_cross_entropy_fwd(const void* logits, const int64_t* targets, float* lse, float* loss, int64_t T, int64_t V,
                           void* stream);
int moss_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse, const float* scale,
                           void* dlogits, int64_t T, int64_t V, void* stream);
/* dq, dk, dv (memory [B, H, S, hd] or, bshd = 1, [B, S, H, hd]) -> dqkv [B, S, 3, H, hd]
 * (inverse rotation) */
int moss_rope_bwd(const void* dq, const void* dk, const void* dv, const float* cosv, const float* sinv, void* dqkv,
                  float* amax, int64_t B, int64_t S, int64_t H, int64_t hd, int bshd, void* stream);


/* ---------------------------------------------------------------------------
 * Per-group (COAT-style) comparator — NOT the MOSS path; the ablation the
 * paper contrasts MOSS with (Fig. 1 / Table 7).
 * quant_per_group (quantize.py:100-124), group = 128 along rows:
 *   scales [rows, cols/128] f32 = f32(amax/448) (0 -> 1), codes = e4m3(x / s) */
int moss_quant_per_group(const void* x, int dtype, int64_t rows, int64_t cols, int64_t group, uint8_t* codes,
                         float* scales, uint32_t* flags, void* stream);
/* gemm_pergroup_mainloop (gemm.py:132-157): D = sum_g (A_g B_g^T) sa[:, g] sb[:, g]^T,
 * every 128-deep partial product rescaled on the CUDA cores ("promotion").
 * Scales GROUP-MAJOR: sa_t [K/128, M], sb_t [K/128, N] f32.  M, N, K % 128 == 0. */
int moss_gemm_pergroup(const uint8_t* A, const float* sa_t, const uint8_t* B, const float* sb_t, void* D,
                       int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, void* stream);

/* Human-readable status. */
const char* moss_strerror(int status);

/* Library ABI version (major*100 + minor). */
int moss_version(void);

#ifdef __cplusplus
}
#endif

#endif /* MOSS_B200_H */
