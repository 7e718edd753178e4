// Layer-wise learn path of fast numerics for MLPs the fused per-tile kernel (kernels_learn.cu,
// widths <= 64 held on chip) cannot hold: every layer is one tcgen05 GEMM over all rows
// (kernels_tgemm.cu) with the activations in HBM as bf16, the reference's
//   forward   Z_l = H_{l-1} W_l + b_l, H_l = act(Z_l)             (ops.cpp:75-106, 28-47, 63-73)
//   backward  dZ_{l-1} = (dZ_l W_l^T) * act'(H_{l-1})             (interp.cpp:392-499, ops.cpp:213-246)
//             dW_l = H_{l-1}^T dZ_l, db_l = column sums of dZ_l  (matmul_grad_rhs, reduce_to_shape)
// with split-K weight-gradient partials in the per-slot layout the fast reduction already sums
// (fixed order: deterministic). This file holds the element-wise pieces around the GEMMs: the
// bf16 weight / input copies, the PPO / A3C / value loss (rl.cpp:137-202) producing dZ_{L-1},
// and the bias-gradient column sums.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "wide.cuh"

namespace flw {

namespace {

// W_l (f32 [din, dout], reference layout) -> bf16 [din, ld] for every layer of both nets.
__global__ void k_wide_weights(const float* __restrict__ params, WideNet n0, __nv_bfloat16* w0, WideNet n1,
                               __nv_bfloat16* w1) {
    const WideNet& n = blockIdx.y == 0 ? n0 : n1;
    __nv_bfloat16* wb = blockIdx.y == 0 ? w0 : w1;
    for (int l = 0; l < n.L; ++l) {
        const int64_t cnt = static_cast<int64_t>(n.din[l]) * n.dout[l];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t r = i / n.dout[l], c = i % n.dout[l];
            wb[n.wofs[l] + r * n.wld[l] + c] = __float2bfloat16(params[n.woff[l] + i]);
        }
    }
}

// row-major f32 [rows, cols] -> bf16 [rows, ld]: one warp per row, consecutive lanes on
// consecutive columns (coalesced both ways, no per-element division)
__global__ void k_wide_to_bf16(const float* __restrict__ x, int64_t rows, int cols, __nv_bfloat16* out, int64_t ld) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
        const float* xr = x + r * cols;
        __nv_bfloat16* orow = out + r * ld;
        for (int c = 2 * lane; c < cols; c += 64) {
            if (c + 1 < cols) {
                const float2 v = make_float2(__ldg(xr + c), __ldg(xr + c + 1));
                if ((ld & 1) == 0)
                    *reinterpret_cast<__nv_bfloat162*>(orow + c) = __floats2bfloat162_rn(v.x, v.y);
                else {
                    orow[c] = __float2bfloat16(v.x);
                    orow[c + 1] = __float2bfloat16(v.y);
                }
            } else {
                orow[c] = __float2bfloat16(__ldg(xr + c));
            }
        }
    }
}

__global__ void k_wide_fill_col(__nv_bfloat16* p, int64_t rows, int64_t ld, int64_t col, float v) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[r * ld + col] = __float2bfloat16(v);
}

__global__ void k_wide_split_input(const float* __restrict__ x, int64_t rows, int cols, __half* out, int64_t seg) {
    const int64_t n = rows * cols;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = i / cols, c = i % cols;
        const float v = x[i];
        const __half hi = __float2half_rn(v);
        __half* o = out + r * 3 * seg + c;
        o[0] = hi;
        o[seg] = __float2half_rn(v - __half2float(hi));
        o[2 * seg] = hi;
    }
}

__global__ void k_wide_split_weights(const float* __restrict__ params, WideNet n, __half* ws) {
    for (int l = 0; l < n.L; ++l) {
        const int64_t cnt = static_cast<int64_t>(n.din[l]) * n.dout[l];
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < cnt;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t r = i / n.dout[l], c = i % n.dout[l];
            const float w = params[n.woff[l] + i];
            const __half hi = __float2half_rn(w);
            __half* o = ws + n.sofs[l] + r * n.wld[l] + c;
            o[0] = hi;                                                        // x_hi . W_hi
            o[n.dp[l] * n.wld[l]] = hi;                                       // x_lo . W_hi
            o[2 * n.dp[l] * n.wld[l]] = __float2half_rn(w - __half2float(hi));  // x_hi . W_lo
        }
    }
}

// One row per thread: the loss terms of rl.cpp:137-202 in f32 (the fused kernel's loss epilogue)
// and dZ_{L-1} rounded to the bf16 operand the backward GEMMs read. Per-block sums of the
// policy / value / entropy terms in a fixed order (block-local tree), one slot per block.
__global__ void __launch_bounds__(256) k_wide_loss(WideLossArgs a) {
    __shared__ float red[3][256];
    float pl = 0.0f, vl = 0.0f, en = 0.0f;
    for (int64_t row = blockIdx.x * 256LL + threadIdx.x; row < a.rows; row += gridDim.x * 256LL) {
        float dz[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) dz[j] = 0.0f;
        const float inv_n = static_cast<float>(a.inv_n);
        if (a.kind == kNetCritic) {  // value MSE: dV = 2 c_v (V - R) / N
            const float verr = a.out[row] - a.ret[row];
            dz[0] = static_cast<float>(2.0 * a.value_coef) * inv_n * verr;
            vl += static_cast<float>(a.value_coef) * inv_n * verr * verr;
        } else {
            const int A = a.A;
            const float* o = a.out + row * A;
            float mx = o[0];
            for (int j = 1; j < A; ++j) mx = fmaxf(mx, o[j]);
            float den = 0.0f;
            for (int j = 0; j < A; ++j) den += __expf(o[j] - mx);
            const float lden = __logf(den);
            float p[16], lp[16], H = 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                lp[j] = j < A ? o[j] - mx - lden : 0.0f;
                p[j] = j < A ? __expf(lp[j]) : 0.0f;
                if (j < A) H -= p[j] * lp[j];
            }
            const int act = a.actions[row];
            float lpa = 0.0f;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j == act) lpa = lp[j];
            float coef;
            if (a.kind == kNetPolicyPpo) {
                float adv = a.adv[row];
                if (a.adv_stats) {
                    const double sd = a.adv_stats[1];
                    if (!(sd < 1e-8)) adv = static_cast<float>((adv - a.adv_stats[0]) / (sd + 1e-8));
                }
                const float ratio = __expf(lpa - a.logp_old[row]);
                const float clipped = fminf(fmaxf(ratio, 1.0f - a.clip_eps), 1.0f + a.clip_eps);
                const float s1 = ratio * adv, s2 = clipped * adv;
                pl -= fminf(s1, s2) * inv_n;
                coef = s1 <= s2 ? -inv_n * ratio * adv : 0.0f;
            } else {  // A3C: advantage R - V (rl.cpp:188)
                const float adv = a.ret[row] - a.values_in[row];
                pl -= lpa * adv * inv_n;
                coef = -inv_n * adv;
            }
            en += H * inv_n;
            const float eci = static_cast<float>(a.entropy_coef) * inv_n;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < A) dz[j] = coef * ((j == act ? 1.0f : 0.0f) - p[j]) + eci * p[j] * (lp[j] + H);
        }
        __nv_bfloat16* d = a.dz + row * a.ld;
        for (int j = 0; j < a.width; ++j) d[j] = __float2bfloat16(dz[j]);
    }
    red[0][threadIdx.x] = pl;
    red[1][threadIdx.x] = vl;
    red[2][threadIdx.x] = en;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x < 3) a.loss_partials[blockIdx.x * 3 + threadIdx.x] = red[threadIdx.x][0];
}

// db partials: part[s * stride + col] = sum of dZ[r, col] over rows r of split s (rows split
// like the weight-gradient GEMM's K range: any fixed split is deterministic). Block = (split,
// 64 columns): 8 threads per row read 16 B each (coalesced 128-byte row segments), 32 row phases;
// the 32 phase sums are added in phase order.
__global__ void __launch_bounds__(256) k_wide_colsum(const __nv_bfloat16* __restrict__ dz, int64_t rows, int cols,
                                                     int64_t ld, int splits, float* part, int64_t stride) {
    __shared__ float red[32][65];
    const int s = blockIdx.x;
    const int c8 = threadIdx.x & 7, ph = threadIdx.x >> 3;
    const int c0 = blockIdx.y * 64 + 8 * c8;
    const int64_t r0 = rows * s / splits, r1 = rows * (s + 1) / splits;
    float acc[8] = {0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f, 0.0f};
    const bool vec = c0 + 8 <= cols && (ld & 7) == 0;
    if (vec) {  // four rows' loads in flight per thread
        int64_t r = r0 + ph;
        for (; r + 96 < r1; r += 128) {
            uint4 u[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) u[k] = __ldg(reinterpret_cast<const uint4*>(dz + (r + 32 * k) * ld + c0));
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u[k]);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f = __bfloat1622float2(h[i]);
                    acc[2 * i] += f.x;
                    acc[2 * i + 1] += f.y;
                }
            }
        }
        for (; r < r1; r += 32) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(dz + r * ld + c0));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(h[i]);
                acc[2 * i] += f.x;
                acc[2 * i + 1] += f.y;
            }
        }
    }
    for (int64_t r = r0 + ph; !vec && r < r1; r += 32) {
        const __nv_bfloat16* p = dz + r * ld + c0;
        if (vec) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 f = __bfloat1622float2(h[i]);
                acc[2 * i] += f.x;
                acc[2 * i + 1] += f.y;
            }
        } else {
            for (int i = 0; i < 8; ++i)
                if (c0 + i < cols) acc[i] += __bfloat162float(p[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) red[ph][8 * c8 + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < 64) {
        const int c = blockIdx.y * 64 + threadIdx.x;
        float t = 0.0f;
        for (int k = 0; k < 32; ++k) t += red[k][threadIdx.x];
        if (c < cols) part[static_cast<int64_t>(s) * stride + c] = t;
    }
}

__global__ void k_wide_sum_partials(const float* __restrict__ part, int splits, int64_t count, float* out) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float t = 0.0f;
        for (int s = 0; s < splits; ++s) t += part[s * count + i];  // split order: deterministic
        out[i] = t;
    }
}

}  // namespace

void wide_sum_partials(cudaStream_t s, const float* part, int splits, int64_t count, float* out) {
    const int blocks = static_cast<int>(std::min<int64_t>((count + 255) / 256, 148 * 8));
    k_wide_sum_partials<<<blocks, 256, 0, s>>>(part, splits, count, out);
}

void wide_build_weights(cudaStream_t s, const float* params, const WideNet& n0, __nv_bfloat16* w0, const WideNet& n1,
                        __nv_bfloat16* w1) {
    k_wide_weights<<<dim3(64, 2), 256, 0, s>>>(params, n0, w0, n1, w1);
}

void wide_to_bf16(cudaStream_t s, const float* x, int64_t rows, int cols, __nv_bfloat16* out, int64_t ld) {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 7) / 8, 148 * 16));
    k_wide_to_bf16<<<blocks, 256, 0, s>>>(x, rows, cols, out, ld);
}

void wide_fill_col(cudaStream_t s, __nv_bfloat16* p, int64_t rows, int64_t ld, int64_t col, float v) {
    const int blocks = static_cast<int>(std::min<int64_t>((rows + 255) / 256, 148 * 8));
    k_wide_fill_col<<<blocks, 256, 0, s>>>(p, rows, ld, col, v);
}

void wide_split_input(cudaStream_t s, const float* x, int64_t rows, int cols, __half* out, int64_t seg) {
    const int64_t n = rows * cols;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 148 * 8));
    k_wide_split_input<<<blocks, 256, 0, s>>>(x, rows, cols, out, seg);
}

void wide_build_split_weights(cudaStream_t s, const float* params, const WideNet& n, __half* ws) {
    k_wide_split_weights<<<64, 256, 0, s>>>(params, n, ws);
}

int wide_loss_blocks(int64_t rows) { return static_cast<int>(std::min<int64_t>(148 * 4, (rows + 255) / 256)); }

void wide_loss(cudaStream_t s, const WideLossArgs& a) {
    k_wide_loss<<<wide_loss_blocks(a.rows), 256, 0, s>>>(a);
}

void wide_colsum(cudaStream_t s, const __nv_bfloat16* dz, int64_t rows, int cols, int64_t ld, int splits, float* part,
                 int64_t stride) {
    k_wide_colsum<<<dim3(splits, (cols + 63) / 64), 256, 0, s>>>(dz, rows, cols, ld, splits, part, stride);
}

}  // namespace flw
