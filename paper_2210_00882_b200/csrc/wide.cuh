// Layer-wise learn path of fast numerics (kernels_wide.cu + the tgemm GEMMs): MLPs wider than
// the fused per-tile kernel's 64 columns (H = 256, SURVEY §8 "also report H=256").
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fast.cuh"

namespace flw {

struct WideNet {
    int L;
    int din[kMaxLayers], dout[kMaxLayers];       // real widths
    int64_t woff[kMaxLayers], boff[kMaxLayers];  // offsets in the flat parameter vector
    int64_t wofs[kMaxLayers], wld[kMaxLayers];   // bf16 weight copy: layer l at wofs, [din, wld]
    int64_t wbytes;                              // elements of the bf16 weight copy
    // rollout (f32-accurate split GEMMs): input segment width dp = din padded to 64, the f16
    // weight image [W_hi; W_hi; W_lo] of layer l at sofs[l], [3 dp, wld] (N contiguous)
    int64_t dp[kMaxLayers], sofs[kMaxLayers];
    int64_t sbytes;
};

struct WideLossArgs {
    int kind;                 // NetKind
    const float* out;         // logits [rows, A] / values [rows]
    int A;
    int64_t rows;
    const int32_t* actions;
    const float *logp_old, *adv, *ret, *values_in;
    const double* adv_stats;  // {mean, sd} or null
    double inv_n, value_coef, entropy_coef;
    float clip_eps;
    __nv_bfloat16* dz;        // dZ_{L-1} [rows, ld] (width columns written)
    int64_t ld;
    int width;
    float* loss_partials;     // [wide_loss_blocks(rows), 3]
};

void wide_build_weights(cudaStream_t s, const float* params, const WideNet& n0, __nv_bfloat16* w0, const WideNet& n1,
                        __nv_bfloat16* w1);
void wide_to_bf16(cudaStream_t s, const float* x, int64_t rows, int cols, __nv_bfloat16* out, int64_t ld);
void wide_fill_col(cudaStream_t s, __nv_bfloat16* p, int64_t rows, int64_t ld, int64_t col, float v);
int wide_loss_blocks(int64_t rows);
// f32 -> f16 hi | lo | hi segments of width seg (x = hi + lo to ~2^-22): the split A operand
void wide_split_input(cudaStream_t s, const float* x, int64_t rows, int cols, __half* out, int64_t seg);
// per layer [W_hi; W_hi; W_lo] f16 (the split B operand)
void wide_build_split_weights(cudaStream_t s, const float* params, const WideNet& n, __half* ws);
void wide_loss(cudaStream_t s, const WideLossArgs& a);
void wide_sum_partials(cudaStream_t s, const float* part, int splits, int64_t count, float* out);  // fixed order
void wide_colsum(cudaStream_t s, const __nv_bfloat16* dz, int64_t rows, int cols, int64_t ld, int splits, float* part,
                 int64_t stride);

}  // namespace flw
