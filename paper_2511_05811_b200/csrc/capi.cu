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
                cudaStream_t st);
int launch_adamw(float* w, const void* g, int g_dtype, float* m, float* v, int64_t rows, int64_t cols,
                 const moss_adam_params& p, float enc_scale, const moss_adam_params* p_dev, const float* enc_dev,
                 float* scale_out, uint8_t* w_fp8, uint8_t* w_fp8_t, float* w_amax, uint32_t* nsat,
                 uint32_t* flags, cudaStream_t st);
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
                   void* stream) {
    if (M <= 0 || N <= 0 || K <= 0) return MOSS_ERR_SHAPE;
    if (K % 128 || M % 128 || N % 128) return MOSS_ERR_SHAPE;
    if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return MOSS_ERR_SHAPE;
    if (!A || !B || !SFA || !sA || !sB || !D || !dtype_ok(d_dtype)) return MOSS_ERR_ARGUMENT;
    if (ldd < N) return MOSS_ERR_SHAPE;
    if (accumulate && d_dtype != MOSS_F32) return MOSS_ERR_ARGUMENT;
    if (!aligned(A, 16) || !aligned(B, 16) || !aligned(SFA, 16) || (SFB && !aligned(SFB, 16)) || !aligned(D, 16) ||
        ldd % 8)
        return MOSS_ERR_ALIGN;
    return moss::launch_gemm(A, SFA, B, SFB, sA, sB, D, d_dtype, ldd, M, N, K, accumulate, (cudaStream_t)stream);
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

}  // extern "C"
