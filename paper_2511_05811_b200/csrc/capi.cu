// extern "C" boundary (include/moss_b200.h).  Host-side argument checks run
// here, before any launch, and map to the reference's exception classes
// (errors.py:4-45) through the status codes.
#include <cstdint>

#include "common.cuh"

namespace moss {
int launch_amax(const void* x, int dtype, int64_t n, float* amax, uint32_t* flags, cudaStream_t st);
int launch_quant_mx2(const void* x, int dtype, int64_t rows, int64_t cols, const float* amax, uint8_t* codes,
                     uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out,
                     uint32_t* flags, cudaStream_t st);
int launch_quant_fused(const void* x, int dtype, int64_t rows, int64_t cols, float* amax, int amax_given,
                       uint8_t* codes, uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                       float* g_out, uint32_t* ws, uint32_t* flags, cudaStream_t st);
int launch_encode_scaled(const void* x, int dtype, int64_t rows, int64_t cols, const float* scale, float scale_host,
                         int from_amax, uint8_t* codes, uint8_t* codes_t, float* scale_out, uint32_t* nsat,
                         uint32_t* flags, cudaStream_t st);
int launch_gemm(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                float* d_amax, uint32_t* flags, cudaStream_t st);
int launch_gemm2_bkn(const uint8_t* A, const uint8_t* SFA, const uint8_t* B_kn, const float* sA, const float* sB,
                     void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, float* d_amax,
                     cudaStream_t st);
int launch_adamw(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                 const moss_adam_params& p, float enc_scale, const moss_adam_params* p_dev, const float* enc_dev,
                 float* scale_out, uint8_t* w_fp8, uint8_t* w_fp8_t, float* w_amax, uint32_t* nsat,
                 uint32_t* flags, cudaStream_t st);
int launch_check_finite(const void* x, int dtype, int64_t n, uint32_t bit, uint32_t* flags, cudaStream_t st);
int launch_rmsnorm_fwd(const void* x, const void* delta, void* x_out, const float* w, float eps, void* y, float* rstd,
                       float* amax, int64_t T, int64_t d, cudaStream_t st);
int launch_rmsnorm_bwd(const void* dy, const void* x, const float* w, const float* rstd, const void* d_res, void* dx,
                       float* dw, float* amax, float* ws, int64_t T, int64_t d, cudaStream_t st);
int64_t rmsnorm_bwd_workspace(int64_t T, int64_t d);
int launch_swiglu_fwd(const void* gu, void* h, float* amax, int64_t T, int64_t f, cudaStream_t st);
int launch_swiglu_bwd(const void* dh, const void* gu, void* dgu, float* amax, int64_t T, int64_t f, cudaStream_t st);
int launch_rope_fwd(const void* qkv, const float* cosv, const float* sinv, void* q, void* k, void* v, int64_t B,
                    int64_t S, int64_t H, int64_t hd, int bshd, cudaStream_t st);
int launch_rope_bwd(const void* dq, const void* dk, const void* dv, const float* cosv, const float* sinv, void* dqkv,
                    float* amax, int64_t B, int64_t S, int64_t H, int64_t hd, int bshd, cudaStream_t st);
int launch_glue(int mode, const void* x, const void* y, const float* scale, float alpha, void* out, float* amax,
                int64_t T, int64_t d, cudaStream_t st);
int launch_sumsq(const void* x, const void* y, int64_t n, float scale, float* acc, float* parts, cudaStream_t st);
int launch_xent_fwd(const void* logits, const int64_t* targets, float* lse, float* loss, int64_t T, int64_t V,
                    cudaStream_t st);
int launch_xent_bwd(const void* logits, const int64_t* targets, const float* lse, const float* scale, void* dlogits,
                    int64_t T, int64_t V, cudaStream_t st);
int launch_quant_per_group(const void* x, int dtype, int64_t rows, int64_t cols, uint8_t* codes, float* scales,
                           uint32_t* flags, cudaStream_t st);
int launch_gemm_pergroup(const uint8_t* A, const float* sa_t, const uint8_t* B, const float* sb_t, void* D,
                         int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, cudaStream_t st);
}  // namespace moss

static inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
static inline bool dtype_ok(int d) { return d == MOSS_F32 || d == MOSS_BF16; }

extern "C" {

int moss_version(void) { return 101; }

int64_t moss_workspace_bytes(void) { return 64; }

const char* moss_strerror(int s) {
    switch (s) {
        case MOSS_OK: return "ok";
        case MOSS_ERR_SHAPE: return "invalid shape";
        case MOSS_ERR_VALUE: return "invalid value";
        case MOSS_ERR_ARGUMENT: return "invalid argument";
        case MOSS_ERR_E8M0: return "e8m0 range";
        case MOSS_ERR_CUDA: return cudaGetErrorString(cudaGetLastError());
        case MOSS_ERR_ALIGN: return "pointer or stride not 16-byte aligned";
        default: return "unknown status";
    }
}

int64_t moss_sf_bytes(int64_t rows, int64_t cols) {
    if (rows <= 0 || cols <= 0 || cols % 32) return -1;
    return ((rows + 127) / 128) * ((cols / 32 + 3) / 4) * 512;
}

int moss_amax(const void* x, int dtype, int64_t n, float* amax, uint32_t* flags, void* stream) {
    if (n <= 0) return MOSS_ERR_SHAPE;
    if (!dtype_ok(dtype) || !amax || !flags || !x) return MOSS_ERR_ARGUMENT;
    if (!aligned(x, 16)) return MOSS_ERR_ALIGN;
    return moss::launch_amax(x, dtype, n, amax, flags, (cudaStream_t)stream);
}

int moss_quant_mx2(const void* x, int dtype, int64_t rows, int64_t cols, const float* amax, uint8_t* codes, uint8_t* sf,
                   uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t, float* g_out, uint32_t* flags,
                   void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 32) return MOSS_ERR_SHAPE;
    const bool col = codes_t || sf_t || micro_t;
    if (col && rows % 32) return MOSS_ERR_SHAPE;
    if (!codes && !sf && !micro && !col) return MOSS_ERR_ARGUMENT;
    if (!dtype_ok(dtype) || !amax || !flags || !x) return MOSS_ERR_ARGUMENT;
    if (!aligned(x, 16) || (codes && !aligned(codes, 8)) || (codes_t && !aligned(codes_t, 16))) return MOSS_ERR_ALIGN;
    return moss::launch_quant_mx2(x, dtype, rows, cols, amax, codes, sf, micro, codes_t, sf_t, micro_t, g_out, flags,
                                  (cudaStream_t)stream);
}

int moss_quant_mx2_fused(const void* x, int dtype, int64_t rows, int64_t cols, float* amax, int amax_given,
                         uint8_t* codes, uint8_t* sf, uint8_t* micro, uint8_t* codes_t, uint8_t* sf_t, uint8_t* micro_t,
                         float* g_out, uint32_t* workspace, uint32_t* flags, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 32) return MOSS_ERR_SHAPE;
    const bool col = codes_t || sf_t || micro_t;
    if (col && rows % 32) return MOSS_ERR_SHAPE;
    if (!codes && !sf && !micro && !col) return MOSS_ERR_ARGUMENT;
    if (!dtype_ok(dtype) || !amax || !flags || !x || !workspace) return MOSS_ERR_ARGUMENT;
    if (!aligned(x, 16) || (codes && !aligned(codes, 8)) || (codes_t && !aligned(codes_t, 16)) ||
        !aligned(workspace, 16))
        return MOSS_ERR_ALIGN;
    return moss::launch_quant_fused(x, dtype, rows, cols, amax, amax_given, codes, sf, micro, codes_t, sf_t, micro_t,
                                    g_out, workspace, flags, (cudaStream_t)stream);
}

int moss_encode_scaled(const void* x, int dtype, int64_t rows, int64_t cols, const float* scale, float scale_host,
                       int scale_from_amax, uint8_t* codes, uint8_t* codes_t, float* scale_out,
                       uint32_t* n_saturated, uint32_t* flags, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 8) return MOSS_ERR_SHAPE;
    if (codes_t && rows % 32) return MOSS_ERR_SHAPE;
    if (!dtype_ok(dtype) || !flags || !x || (!codes && !codes_t && !scale_out)) return MOSS_ERR_ARGUMENT;
    if (!scale && !(scale_host > 0.f)) return MOSS_ERR_VALUE;
    if (!aligned(x, 16) || (codes && !aligned(codes, 8)) || (codes_t && !aligned(codes_t, 16))) return MOSS_ERR_ALIGN;
    return moss::launch_encode_scaled(x, dtype, rows, cols, scale, scale_host, scale_from_amax, codes, codes_t,
                                      scale_out, n_saturated, flags, (cudaStream_t)stream);
}

int moss_gemm_mxf8(const uint8_t* A, const uint8_t* SFA, const uint8_t* B, const uint8_t* SFB, const float* sA,
                   const float* sB, void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, int accumulate,
                   float* d_amax, uint32_t* flags, void* stream) {
    if (M <= 0 || N <= 0 || K <= 0) return MOSS_ERR_SHAPE;
    if (K % 128 || M % 128 || N % 128) return MOSS_ERR_SHAPE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!A || !B || !SFA || !sA || !sB || !D || !dtype_ok(d_dtype)) return MOSS_ERR_ARGUMENT;
    if (ldd < N) return MOSS_ERR_SHAPE;
    if (accumulate && d_dtype != MOSS_F32) return MOSS_ERR_ARGUMENT;
    if (d_amax && (accumulate || ldd != N || !flags)) return MOSS_ERR_ARGUMENT;
    if (!aligned(A, 16) || !aligned(B, 16) || !aligned(SFA, 16) || (SFB && !aligned(SFB, 16)) || !aligned(D, 16) ||
        ldd % 8)
        return MOSS_ERR_ALIGN;
    return moss::launch_gemm(A, SFA, B, SFB, sA, sB, D, d_dtype, ldd, M, N, K, accumulate, d_amax, flags,
                             (cudaStream_t)stream);
}

int moss_gemm_mxf8_bkn(const uint8_t* A, const uint8_t* SFA, const uint8_t* B_kn, const float* sA, const float* sB,
                       void* D, int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, float* d_amax,
                       void* stream) {
    if (M <= 0 || N <= 0 || K <= 0) return MOSS_ERR_SHAPE;
    if (K % 128 || M % 256 || N % 256) return MOSS_ERR_SHAPE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!A || !B_kn || !SFA || !sA || !sB || !D || !dtype_ok(d_dtype)) return MOSS_ERR_ARGUMENT;
    if (ldd < N) return MOSS_ERR_SHAPE;
    if (!aligned(A, 16) || !aligned(B_kn, 16) || !aligned(SFA, 16) || !aligned(D, 16) || ldd % 8) return MOSS_ERR_ALIGN;
    return moss::launch_gemm2_bkn(A, SFA, B_kn, sA, sB, D, d_dtype, ldd, M, N, K, d_amax, (cudaStream_t)stream);
}

int moss_adamw_fp8(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                   const moss_adam_params* p, float enc_scale, uint8_t* w_fp8, uint8_t* w_fp8_t, float* w_amax,
                   uint32_t* n_saturated, uint32_t* flags, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 8) return MOSS_ERR_SHAPE;
    if (w_fp8_t && rows % 32) return MOSS_ERR_SHAPE;
    if (!w || !g || !m || !v || !p || !flags || !dtype_ok(g_dtype)) return MOSS_ERR_ARGUMENT;
    if ((w_fp8 || w_fp8_t) && !(enc_scale > 0.f)) return MOSS_ERR_VALUE;
    if (!(p->bc1 > 0.f) || !(p->bc2 > 0.f)) return MOSS_ERR_ARGUMENT;
    if (!aligned(w, 16) || !aligned(g, 16) || !aligned(m, 16) || !aligned(v, 16) || (w_fp8 && !aligned(w_fp8, 8)) ||
        (w_fp8_t && !aligned(w_fp8_t, 16)))
        return MOSS_ERR_ALIGN;
    return moss::launch_adamw(w, g, g_dtype, m, v, rows, cols, *p, enc_scale, nullptr, nullptr, nullptr, w_fp8,
                              w_fp8_t, w_amax, n_saturated, flags, (cudaStream_t)stream);
}

int moss_adamw_fp8_dev(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                       const moss_adam_params* p_dev, const float* enc_scale_dev, float* scale_out, uint8_t* w_fp8,
                       uint8_t* w_fp8_t, float* w_amax, uint32_t* n_saturated, uint32_t* flags, void* stream) {
    if (rows <= 0 || cols <= 0 || cols % 8) return MOSS_ERR_SHAPE;
    if (w_fp8_t && rows % 32) return MOSS_ERR_SHAPE;
    if (!w || !g || !m || !v || !p_dev || !flags || !dtype_ok(g_dtype)) return MOSS_ERR_ARGUMENT;
    if ((w_fp8 || w_fp8_t || scale_out) && !enc_scale_dev) return MOSS_ERR_ARGUMENT;
    if (!aligned(w, 16) || !aligned(g, 16) || !aligned(m, 16) || !aligned(v, 16) || !aligned(p_dev, 4) ||
        (w_fp8 && !aligned(w_fp8, 8)) || (w_fp8_t && !aligned(w_fp8_t, 16)))
        return MOSS_ERR_ALIGN;
    moss_adam_params dummy{};
    return moss::launch_adamw(w, g, g_dtype, m, v, rows, cols, dummy, 1.0f, p_dev, enc_scale_dev, scale_out, w_fp8,
                              w_fp8_t, w_amax, n_saturated, flags, (cudaStream_t)stream);
}

int moss_check_finite(const void* x, int dtype, int64_t n, uint32_t bit, uint32_t* flags, void* stream) {
    if (n < 0) return MOSS_ERR_SHAPE;
    if (!x || !flags || !dtype_ok(dtype) || !bit) return MOSS_ERR_ARGUMENT;
    if (!aligned(x, 16)) return MOSS_ERR_ALIGN;
    return moss::launch_check_finite(x, dtype, n, bit, flags, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- producer kernels (bf16)
static inline bool al16(const void* p) { return p == nullptr || aligned(p, 16); }

int moss_rmsnorm_fwd(const void* x, const void* delta, void* x_out, const float* w, float eps, void* y, float* rstd,
                     float* amax, int64_t T, int64_t d, void* stream) {
    if (T <= 0 || d <= 0 || d % 8 || d > 8192 || T > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!x || !w || !y || !rstd || (delta && !x_out)) return MOSS_ERR_ARGUMENT;
    if (!al16(x) || !al16(delta) || !al16(x_out) || !al16(w) || !al16(y)) return MOSS_ERR_ALIGN;
    return moss::launch_rmsnorm_fwd(x, delta, x_out, w, eps, y, rstd, amax, T, d, (cudaStream_t)stream);
}

int64_t moss_rmsnorm_bwd_workspace_bytes(int64_t T, int64_t d) {
    if (T <= 0 || d <= 0 || d % 8 || d > 8192) return -1;
    return moss::rmsnorm_bwd_workspace(T, d);
}

int moss_rmsnorm_bwd(const void* dy, const void* x, const float* w, const float* rstd, const void* d_res, void* dx,
                     float* dw, float* amax, float* workspace, int64_t T, int64_t d, void* stream) {
    if (T <= 0 || d <= 0 || d % 8 || d > 8192 || T > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!dy || !x || !w || !rstd || !dx || (dw && !workspace)) return MOSS_ERR_ARGUMENT;
    if (!al16(dy) || !al16(x) || !al16(w) || !al16(d_res) || !al16(dx) || !al16(dw) || !al16(workspace))
        return MOSS_ERR_ALIGN;
    return moss::launch_rmsnorm_bwd(dy, x, w, rstd, d_res, dx, dw, amax, workspace, T, d, (cudaStream_t)stream);
}

int moss_swiglu_fwd(const void* gu, void* h, float* amax, int64_t T, int64_t f, void* stream) {
    if (T <= 0 || f <= 0 || f % 8) return MOSS_ERR_SHAPE;
    if (!gu || !h) return MOSS_ERR_ARGUMENT;
    if (!al16(gu) || !al16(h)) return MOSS_ERR_ALIGN;
    return moss::launch_swiglu_fwd(gu, h, amax, T, f, (cudaStream_t)stream);
}

int moss_swiglu_bwd(const void* dh, const void* gu, void* dgu, float* amax, int64_t T, int64_t f, void* stream) {
    if (T <= 0 || f <= 0 || f % 8) return MOSS_ERR_SHAPE;
    if (!dh || !gu || !dgu) return MOSS_ERR_ARGUMENT;
    if (!al16(dh) || !al16(gu) || !al16(dgu)) return MOSS_ERR_ALIGN;
    return moss::launch_swiglu_bwd(dh, gu, dgu, amax, T, f, (cudaStream_t)stream);
}

int moss_rope_fwd(const void* qkv, const float* cosv, const float* sinv, void* q, void* k, void* v, int64_t B,
                  int64_t S, int64_t H, int64_t hd, int bshd, void* stream) {
    if (B <= 0 || S <= 0 || H <= 0 || hd <= 0 || hd % 8) return MOSS_ERR_SHAPE;
    if (!qkv || !cosv || !sinv || !q || !k || !v) return MOSS_ERR_ARGUMENT;
    if (!al16(qkv) || !al16(cosv) || !al16(sinv) || !al16(q) || !al16(k) || !al16(v)) return MOSS_ERR_ALIGN;
    return moss::launch_rope_fwd(qkv, cosv, sinv, q, k, v, B, S, H, hd, bshd != 0, (cudaStream_t)stream);
}

int moss_rope_bwd(const void* dq, const void* dk, const void* dv, const float* cosv, const float* sinv, void* dqkv,
                  float* amax, int64_t B, int64_t S, int64_t H, int64_t hd, int bshd, void* stream) {
    if (B <= 0 || S <= 0 || H <= 0 || hd <= 0 || hd % 8) return MOSS_ERR_SHAPE;
    if (!dq || !dk || !dv || !cosv || !sinv || !dqkv) return MOSS_ERR_ARGUMENT;
    if (!al16(dq) || !al16(dk) || !al16(dv) || !al16(cosv) || !al16(sinv) || !al16(dqkv)) return MOSS_ERR_ALIGN;
    return moss::launch_rope_bwd(dq, dk, dv, cosv, sinv, dqkv, amax, B, S, H, hd, bshd != 0, (cudaStream_t)stream);
}

int moss_glue(int mode, const void* x, const void* y, const float* scale, float alpha, void* out, float* amax,
              int64_t T, int64_t d, void* stream) {
    if (T <= 0 || d <= 0 || d % 8 || mode < 0 || mode > 3) return mode < 0 || mode > 3 ? MOSS_ERR_ARGUMENT : MOSS_ERR_SHAPE;
    if (!x || !out || (mode == 2 && !y) || (mode == 3 && !scale)) return MOSS_ERR_ARGUMENT;
    if (!al16(x) || !al16(y) || !al16(out)) return MOSS_ERR_ALIGN;
    return moss::launch_glue(mode, x, y, scale, alpha, out, amax, T, d, (cudaStream_t)stream);
}

int moss_sumsq(const void* x, const void* y, int64_t n, float scale, float* acc, float* partials, void* stream) {
    if (n <= 0 || n % 8) return MOSS_ERR_SHAPE;
    if (!x || !acc || !partials) return MOSS_ERR_ARGUMENT;
    if (!al16(x) || !al16(y)) return MOSS_ERR_ALIGN;
    return moss::launch_sumsq(x, y, n, scale, acc, partials, (cudaStream_t)stream);
}

int moss_cross_entropy_fwd(const void* logits, const int64_t* targets, float* lse, float* loss, int64_t T, int64_t V,
                           void* stream) {
    if (T <= 0 || V <= 0 || V % 8 || T > INT32_MAX || V > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!logits || !targets || !lse || !loss) return MOSS_ERR_ARGUMENT;
    if (!al16(logits)) return MOSS_ERR_ALIGN;
    return moss::launch_xent_fwd(logits, targets, lse, loss, T, V, (cudaStream_t)stream);
}

int moss_cross_entropy_bwd(const void* logits, const int64_t* targets, const float* lse, const float* scale,
                           void* dlogits, int64_t T, int64_t V, void* stream) {
    if (T <= 0 || V <= 0 || V % 8 || T > INT32_MAX || V > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!logits || !targets || !lse || !scale || !dlogits) return MOSS_ERR_ARGUMENT;
    if (!al16(logits) || !al16(dlogits)) return MOSS_ERR_ALIGN;
    return moss::launch_xent_bwd(logits, targets, lse, scale, dlogits, T, V, (cudaStream_t)stream);
}

// ---------------------------------------------------------------- per-group comparator (COAT-style)
int moss_quant_per_group(const void* x, int dtype, int64_t rows, int64_t cols, int64_t group, uint8_t* codes,
                         float* scales, uint32_t* flags, void* stream) {
    if (rows <= 0 || cols <= 0) return MOSS_ERR_SHAPE;
    if (group != 128) return MOSS_ERR_ARGUMENT;             /* the comparator's group size */
    if (cols % 128) return MOSS_ERR_SHAPE;
    if (!x || !codes || !scales || !flags || !dtype_ok(dtype)) return MOSS_ERR_ARGUMENT;
    if (!aligned(x, 16) || !aligned(codes, 4) || !aligned(scales, 4)) return MOSS_ERR_ALIGN;
    return moss::launch_quant_per_group(x, dtype, rows, cols, codes, scales, flags, (cudaStream_t)stream);
}

int moss_gemm_pergroup(const uint8_t* A, const float* sa_t, const uint8_t* B, const float* sb_t, void* D,
                       int d_dtype, int64_t ldd, int64_t M, int64_t N, int64_t K, void* stream) {
    if (M <= 0 || N <= 0 || K <= 0 || M % 128 || N % 128 || K % 128) return MOSS_ERR_SHAPE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || ldd < N) return MOSS_ERR_SHAPE;
    if (!A || !B || !sa_t || !sb_t || !D || !dtype_ok(d_dtype)) return MOSS_ERR_ARGUMENT;
    if (!aligned(A, 16) || !aligned(B, 16) || !aligned(sa_t, 16) || !aligned(sb_t, 16) || !aligned(D, 16) || ldd % 8)
        return MOSS_ERR_ALIGN;
    return moss::launch_gemm_pergroup(A, sa_t, B, sb_t, D, d_dtype, ldd, M, N, K, (cudaStream_t)stream);
}

}  // extern "C"
