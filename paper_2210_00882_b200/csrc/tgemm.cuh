// Generic warp-specialised tcgen05 GEMM over row-major global tensors (kernels_tgemm.cu):
//
//     D[M x N] (f32, TMEM) = op(A)[M x K] * op(B)[K x N]     per (128-row tile, BN-column tile,
//                                                             K split), then a fused epilogue
//
// Operands are loaded by TMA (cp.async.bulk.tensor.2d, 128-byte swizzle) straight from
// row-major global memory, so the layer-wise learn path (H > 64, wide MAPPO inputs) needs no
// operand images:
//   A K-major : stored [M rows, K cols]      (activations H, dZ)
//   A MN-major: stored [K rows, M cols]      (H^T of the weight-gradient GEMM dW = H^T dZ)
//   B K-major : stored [N rows, K cols]      (W as [din, dout] for dH = dZ W^T)
//   B MN-major: stored [K rows, N cols]      (W as [din, dout] for Z = H W; dZ for dW)
// Element types: bf16 (kind::f16) or f32 read as tf32 (kind::tf32; K-major A and B only). Out-of-range rows / cols
// of a box are zero-filled by the TMA unit, so ragged M, N, K need no padding in memory (only
// 16-byte aligned row strides).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace flw {

enum TgType : int { kTgBF16 = 0, kTgF16 = 1, kTgF32 = 2 };  // f32 operands are read as tf32

enum TgEpi : int {
    kTgStoreF32 = 0,    // C32[m, n] = acc (split s at C32 + s * split_stride): split-K partials
    kTgBiasAct = 1,     // C16[m, n] = bf16(act(acc + bias[n])) (and C32 if set)
    kTgBias = 2,        // C32[m, n] = acc + bias[n]
    kTgActGrad = 3,     // C16[m, n] = bf16(acc * act'(H[m, n])), H bf16 (act' from the output)
    kTgSplit3 = 4,      // y = act(acc + bias[n]) (accurate tanhf), written as f16 hi | lo | hi
                        // (y = hi + lo): the next layer's A operand of the split f32-accurate GEMM
};

struct TgOperand {
    const void* ptr;
    int64_t rows, cols, ld;  // storage [rows, cols] row-major, ld in elements (ld * esz % 16 == 0)
    int dt;                  // TgType
};

struct TgEpilogue {
    int mode = kTgStoreF32;
    int act = 0;                        // 0 tanh, 1 relu
    float* c32 = nullptr;
    int64_t ldc32 = 0;
    int64_t split_stride = 0;           // elements between the partials of consecutive K splits
    __nv_bfloat16* c16 = nullptr;
    int64_t ldc16 = 0;
    const float* bias = nullptr;        // [N]
    const __nv_bfloat16* h = nullptr;   // kTgActGrad: activation whose derivative scales acc
    int64_t ldh = 0;
    int64_t m_store = -1, n_store = -1; // stored extent (default M, N)
    __half* c16h = nullptr;             // kTgSplit3: [m, seg*k + n] for the segments hi, lo, hi
    int64_t seg = 0;
};

// D = op(A) op(B) with K split `splits` ways (kTgStoreF32 only for splits > 1). bn: 64, 128 or
// 256 (the N tile). grid_cap: max CTAs (0: one per SM).
void tgemm(cudaStream_t s, const TgOperand& A, bool a_mn, const TgOperand& B, bool b_mn, int64_t M, int64_t N,
           int64_t K, int splits, const TgEpilogue& epi, int bn = 128, int grid_cap = 0);

}  // namespace flw
