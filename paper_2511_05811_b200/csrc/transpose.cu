// Byte-matrix transpose: dst [cols, rows] = src [rows, cols]^T (u8).
//
// Used by the ZeRO-1 path (zero.py): after the FP8 all-gather of a weight's
// row-major E4M3 codes W_fp8 [out, in], each rank rebuilds the dgrad operand
// W_fp8^T [in, out] locally (1 B read + 1 B written per parameter) instead of
// gathering a column-sharded transpose.  Per-tensor codes commute with the
// transpose, so this equals encoding W^T directly.
//
// 64 x 64 byte tiles through shared memory: 16-byte loads of 64-byte row
// segments, 16-byte stores of 64-byte column segments.
#include "common.cuh"

namespace moss {

constexpr int TR_T = 64;

__global__ void __launch_bounds__(256) transpose_u8_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                                           int64_t rows, int64_t cols) {
    __shared__ uint8_t tile[TR_T][TR_T + 4];
    const int tid = threadIdx.x;
    const int64_t r0 = (int64_t)blockIdx.y * TR_T, c0 = (int64_t)blockIdx.x * TR_T;
    {   // load: thread -> (row tid/4, 16-byte chunk tid%4)
        const int r = tid >> 2, ch = (tid & 3) * 16;
        const int64_t gr = r0 + r, gc = c0 + ch;
        uint8_t b[16];
        if (gr < rows && gc + 16 <= cols) {
            const uint4 u = *reinterpret_cast<const uint4*>(src + gr * cols + gc);
            *reinterpret_cast<uint4*>(b) = u;
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) b[i] = (gr < rows && gc + i < cols) ? src[gr * cols + gc + i] : 0;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) tile[r][ch + i] = b[i];
    }
    __syncthreads();
    {   // store: thread -> (output row = input column tid/4, 16 input rows starting at (tid%4)*16)
        const int c = tid >> 2, rs = (tid & 3) * 16;
        const int64_t orow = c0 + c, ocol = r0 + rs;
        uint8_t b[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) b[i] = tile[rs + i][c];
        if (orow < cols && ocol + 16 <= rows) {
            *reinterpret_cast<uint4*>(dst + orow * rows + ocol) = *reinterpret_cast<const uint4*>(b);
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if (orow < cols && ocol + i < rows) dst[orow * rows + ocol + i] = b[i];
        }
    }
}

int launch_transpose_u8(const uint8_t* src, uint8_t* dst, int64_t rows, int64_t cols, cudaStream_t st) {
    dim3 grid((unsigned)((cols + TR_T - 1) / TR_T), (unsigned)((rows + TR_T - 1) / TR_T));
    transpose_u8_kernel<<<grid, 256, 0, st>>>(src, dst, rows, cols);
    return cudaPeekAtLastError() == cudaSuccess ? MOSS_OK : MOSS_ERR_CUDA;
}

}  // namespace moss
