// Fast-numerics learn phase: the whole PPO/A3C train iteration of one MLP fused per 128-row
// tile on the 5th-gen tensor cores.
//
//   critic forward  (mode 0): values / last_value for GAE
//   learn           (mode 1): forward (L layers) -> loss epilogue -> backward (L layers), with
//                             dW_l += H_{l-1}^T dZ_l accumulated in TMEM across all tiles a CTA
//                             owns, db_l by column sums, per-CTA partials written once at the end.
//
// One CTA per SM (persistent, grid = #SMs), 256 threads: warp w reads TMEM lane quadrant w%4,
// so rows r = 32*(w%4) + lane are shared by warps w and w+4, which split each row's columns
// (16-column chunks alternate between the two halves). Thread 0 issues tcgen05.mma. Operands are
// bf16 in shared memory in the core-matrix layout of umma.cuh; activations H_l written once
// serve as the K-major A of the next forward GEMM and as the MN-major A of the dW GEMM.
// Accumulation is f32 (TMEM).
// TMEM map (512 columns): [0,64) = Z (M=128 forward / dH accumulator); layer pair (2j, 2j+1)
// dW accumulators (M=64, "half sub-partition" layout) share columns [64+64j, 128+64j) at
// lane offsets 0 and 16.
#include <cuda_runtime.h>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"
#include "engine.hpp"
#include "fast.cuh"
#include "umma.cuh"
#include "update.cuh"

namespace flw {

namespace {

constexpr int kRows = 128;

struct Smem {  // the weight image of one net (byte offsets; k_learn's shared-memory prefix)
    uint32_t wt[kMaxLayers], x, hbytes;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem carve(const FastNet& n) {
    Smem s{};
    uint32_t off = 0;
    for (int l = 0; l < n.L; ++l) {
        s.wt[l] = off;
        off = align_up(off + static_cast<uint32_t>(n.dout[l] * n.din[l] * 2), 128);
    }
    s.x = off;  // end of the weight image
    s.hbytes = static_cast<uint32_t>(kRows * n.din[0] * 2);  // the input tile X, then H_0 .. H_{L-2}
    for (int l = 0; l + 1 < n.L; ++l) s.hbytes += static_cast<uint32_t>(kRows * n.dout[l] * 2);
    return s;
}

// Weight-tile image: W_l^T as [dout x din] K-major bf16 core-matrix tiles, zero padded, at the
// offsets carve() assigns; k_learn copies it into the front of its shared memory once per CTA.
__global__ void __launch_bounds__(256) k_build_wimg(const float* __restrict__ params, FastNet n0,
                                                    __nv_bfloat16* __restrict__ img0, FastNet n1,
                                                    __nv_bfloat16* __restrict__ img1) {
    const FastNet& n = blockIdx.y == 0 ? n0 : n1;  // blockIdx.y: which net (both in one launch)
    __nv_bfloat16* img = blockIdx.y == 0 ? img0 : img1;
    const Smem S = carve(n);
    for (int l = 0; l < n.L; ++l) {
        const int di = n.din[l], dout = n.dout[l], ri = n.rin[l], ro = n.rout[l];
        const float* W = params + n.woff[l];
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < dout * di; i += gridDim.x * blockDim.x) {
            const int o = i / di, c = i % di;
            const float v = (o < ro && c < ri) ? W[c * ro + o] : 0.0f;
            img[(S.wt[l] + umma::tile_offset(o, c, di)) / 2] = __float2bfloat16(v);
        }
    }
}

// ------------------------------------------------------------------ partial reduction
// grads[p] = sum over CTA partials in CTA order (deterministic); both nets in one launch, the
// critic's partials following the policy's in the flat gradient.
__global__ void __launch_bounds__(256) k_reduce_partials(const float* __restrict__ pp, const float* __restrict__ pc,
                                                         int np, int nc, int64_t Pp, int64_t Pc, int64_t c_off,
                                                         float* grads) {
    // 32 parameters per block (lane = parameter, coalesced rows); warp w sums partials
    // w, w+8, ... in order, then the 8 warp sums are added in warp order: a fixed tree.
    __shared__ float ws[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * 32LL + lane;
    const bool ok = i < Pp + Pc;
    const float* src = !ok ? pp : (i < Pp ? pp + i : pc + (i - Pp));
    const int64_t stride = i < Pp ? Pp : Pc;
    const int nparts = i < Pp ? np : nc;
    float s = 0.0f;
    if (ok) {
#pragma unroll 8
        for (int p = w; p < nparts; p += 8) s += src[p * stride];  // loads hoisted, adds in order
    }
    ws[w][lane] = s;
    __syncthreads();
    if (w == 0 && ok) {
        float t = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += ws[k][lane];
        grads[i < Pp ? i : i + c_off] = t;
    }
}

// One train iteration's parameter update fused into a single launch (1 GPU, no exchange): the
// fixed-order reduction of the per-CTA dW partials (as k_reduce_partials), Adam with double
// moments (mlp.cpp:146-161, as k_adam) and the bf16 weight-image entry of every weight (as
// k_build_wimg), so the next train iteration's learn kernels read the updated image without a
// build launch. The Adam step counter and its bias corrections (as k_adam_tick) are advanced by
// the last block to finish (every block has read the old counter by then).
// kPdl: launched as a programmatic dependent of the learn kernel (k_learn triggers its
// dependents when its tiles are done): the Adam operands are fetched before the wait.
template <bool kPdl>
__global__ void __launch_bounds__(256) k_reduce_adam(FastUpdateArgs a, int nchunks) {
    __shared__ float4 ws[8][32];
    int64_t t;
    double bc1, bc2;
    adam_step_consts(a, t, bc1, bc2);
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x)
        update_chunk<12, kPdl>(a, c, threadIdx.x, ws, bc1, bc2, [] { __syncthreads(); });
    if constexpr (kPdl)
        if (blockIdx.x >= nchunks) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) update_arrive(a, t, bc1, bc2, gridDim.x);
}

__global__ void k_reduce_loss(const float* __restrict__ lp, int np, int nc, double ec, float* loss) {
    const int lane = threadIdx.x;
    double pl = 0, vl = 0, en = 0;
    for (int p = lane; p < np + nc; p += 32) {  // policy slots [0, np), critic slots [np, np + nc)
        const float* q = lp + p * 3;
        pl += q[0];
        vl += q[1];
        en += q[2];
    }
    for (int off = 16; off > 0; off >>= 1) {
        pl += __shfl_xor_sync(0xffffffffu, pl, off);
        vl += __shfl_xor_sync(0xffffffffu, vl, off);
        en += __shfl_xor_sync(0xffffffffu, en, off);
    }
    if (lane == 0) *loss = static_cast<float>(pl + vl - ec * en);
}

// --------------------------------------------------------------------- GAE (parallel)
// Thread per stream (rl.cpp:28-95 recurrences in double); the T-loop is processed in chunks of 8
// steps whose loads are issued together. Per-block sums of adv and adv^2 feed the normalisation
// statistics, combined in fixed block order by k_adv_stats.
template <int CH, int MINB>
__global__ void __launch_bounds__(256, MINB) k_fast_gae(const float* __restrict__ rew, const float* __restrict__ values,
                                                  const float* __restrict__ done_f,
                                                  const float* __restrict__ last_value, int64_t T, int64_t R,
                                                  double gamma, double lam, float* adv, float* ret, bool with_adv,
                                                  double* block_sums, double* stats, unsigned* done_counter) {
    __shared__ double s1[256], s2[256];
    int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    double a1 = 0.0, a2 = 0.0;
    if (s < R) {
        const double gl = gamma * lam;
        const double lv = last_value[s];
        double acc = 0.0, running = lv, next_v = lv;
        for (int64_t hi = T - 1; hi >= 0; hi -= CH) {
            float rr[CH], vv[CH], dd[CH];
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                int64_t tt = hi - j;
                if (tt >= 0) {
                    int64_t i = tt * R + s;
                    rr[j] = rew[i];
                    vv[j] = values[i];
                    dd[j] = done_f[i];
                }
            }
#pragma unroll
            for (int j = 0; j < CH; ++j) {
                int64_t tt = hi - j;
                if (tt < 0) break;
                int64_t i = tt * R + s;
                const bool done = dd[j] > 0.5f;
                const double r = rr[j], v = vv[j];
                if (with_adv) {
                    double nv = done ? 0.0 : next_v;
                    if (done) acc = 0.0;
                    acc = (r + gamma * nv - v) + gl * acc;
                    adv[i] = static_cast<float>(acc);
                    a1 += acc;
                    a2 += acc * acc;
                }
                next_v = v;
                if (done) running = 0.0;
                running = r + gamma * running;
                ret[i] = static_cast<float>(running);
            }
        }
    }
    s1[threadIdx.x] = a1;
    s2[threadIdx.x] = a2;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        block_sums[2 * blockIdx.x] = s1[0];
        block_sums[2 * blockIdx.x + 1] = s2[0];
    }
    if (!done_counter || !with_adv) return;
    // the last block to finish combines the block sums (fixed block order -> deterministic)
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    a1 = 0.0;
    a2 = 0.0;
    for (int b = threadIdx.x; b < static_cast<int>(gridDim.x); b += 256) {
        a1 += __ldcg(block_sums + 2 * b);
        a2 += __ldcg(block_sums + 2 * b + 1);
    }
    s1[threadIdx.x] = a1;
    s2[threadIdx.x] = a2;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double n = static_cast<double>(T * R);
        const double mean = s1[0] / n;
        const double var = s2[0] / n - mean * mean;
        stats[0] = mean;
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
        *done_counter = 0;  // ready for the next launch
    }
}

// Fixed-order (deterministic) parallel combine of the per-block sums: strided partials per
// thread, then a shared-memory tree.
__global__ void __launch_bounds__(256) k_adv_stats(const double* __restrict__ block_sums, int nblocks, int64_t n,
                                                   double* stats) {
    __shared__ double s1[256], s2[256];
    double a1 = 0.0, a2 = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += 256) {
        a1 += block_sums[2 * b];
        a2 += block_sums[2 * b + 1];
    }
    s1[threadIdx.x] = a1;
    s2[threadIdx.x] = a2;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) {
            s1[threadIdx.x] += s1[threadIdx.x + off];
            s2[threadIdx.x] += s2[threadIdx.x + off];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double mean = s1[0] / static_cast<double>(n);
        const double var = s2[0] / static_cast<double>(n) - mean * mean;
        stats[0] = mean;
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

// Warp-shuffle reverse scan (T = 32, the reference default): one block = 32 streams x 32 steps.
// The [T][R] tile is staged through shared memory (coalesced rows), then warp w owns stream w
// with lane = step t. Both recurrences are affine, x_t = b_t + a_t x_{t+1} (rl.cpp:28-47, 66-79:
// GAE a_t = (1 - done_t) gamma lambda, returns a_t = (1 - done_t) gamma), so a 5-step shuffle
// scan of (a, b) pairs replaces the 32-step chain. Double precision, like the sequential kernel.
__device__ __forceinline__ void rscan_affine(double& a, double& b, int lane) {
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const double an = __shfl_down_sync(0xffffffffu, a, off);
        const double bn = __shfl_down_sync(0xffffffffu, b, off);
        if (lane + off < 32) {
            b = b + a * bn;
            a = a * an;
        }
    }
}

__global__ void __launch_bounds__(1024) k_gae_scan32(const float* __restrict__ rew, const float* __restrict__ values,
                                                     const float* __restrict__ done_f,
                                                     const float* __restrict__ last_value, int64_t R, double gamma,
                                                     double lam, float* adv, float* ret, bool with_adv,
                                                     double* block_sums, double* stats, unsigned* done_counter,
                                                     bool pdl) {
    if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");  // the values pass's output
    // Persistent over tiles of 32 streams x 32 steps (grid-stride); the next tile's inputs are
    // loaded into registers while the current one is scanned, so the loads of consecutive tiles
    // overlap (bandwidth regime) and a single tile per block is the latency regime of C2.
    __shared__ float sr[32][33], sv[32][33], sd[32][33];
    __shared__ double w1[32], w2[32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t ntile = (R + 31) / 32;
    float pr = 0.0f, pv = 0.0f, pd = 1.0f, plv = 0.0f;
    auto fetch = [&](int64_t tile) {  // coalesced: warp w loads step t = w of the tile's 32 streams
        const int64_t s0 = tile * 32;
        const int64_t i = static_cast<int64_t>(w) * R + s0 + lane;
        const bool ok = s0 + lane < R;
        pr = ok ? rew[i] : 0.0f;
        pv = ok ? values[i] : 0.0f;
        pd = ok ? done_f[i] : 1.0f;
        plv = s0 + w < R ? last_value[s0 + w] : 0.0f;  // this warp's stream (broadcast)
    };
    double a1 = 0.0, a2 = 0.0;  // this lane's advantage sums, tiles in order
    if (blockIdx.x < ntile) fetch(blockIdx.x);
    for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x) {
        const int64_t s0 = tile * 32;
        __syncthreads();  // the previous tile's transposed outputs were read
        sr[w][lane] = pr;
        sv[w][lane] = pv;
        sd[w][lane] = pd;
        const float lvf = plv;
        __syncthreads();
        if (tile + gridDim.x < ntile) fetch(tile + gridDim.x);  // prefetch the next tile
        const int64_t st = s0 + w;  // this warp's stream; lane = step t
        const bool live = st < R;
        const int t = lane;
        const bool done = sd[t][w] > 0.5f;
        const double r = sr[t][w], v = sv[t][w];
        const double lv = live ? static_cast<double>(lvf) : 0.0;
        const double vnext = t == 31 ? lv : static_cast<double>(sv[t + 1][w]);
        // GAE: acc_t = delta_t + (done_t ? 0 : gamma lambda) acc_{t+1}, acc_32 = 0
        double a = done ? 0.0 : gamma * lam;
        double b = (r + gamma * (done ? 0.0 : vnext)) - v;
        rscan_affine(a, b, lane);
        const double acc = b;  // + a * 0
        // returns: run_t = r_t + (done_t ? 0 : gamma) run_{t+1}, run_32 = last_value
        double ar = done ? 0.0 : gamma, br = r;
        rscan_affine(ar, br, lane);
        const double run = br + ar * lv;
        __syncthreads();
        sr[t][w] = static_cast<float>(run);  // reuse the tiles for the transposed stores
        sv[t][w] = static_cast<float>(acc);
        if (live && with_adv) {
            a1 += acc;
            a2 += acc * acc;
        }
        __syncthreads();
        const int64_t i = static_cast<int64_t>(w) * R + s0 + lane;
        if (s0 + lane < R) {
            ret[i] = sr[w][lane];
            if (with_adv) adv[i] = sv[w][lane];
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        a1 += __shfl_xor_sync(0xffffffffu, a1, off);
        a2 += __shfl_xor_sync(0xffffffffu, a2, off);
    }
    if (lane == 0) {
        w1[w] = a1;
        w2[w] = a2;
    }
    __syncthreads();
    if (w == 0) {  // block sums in warp order, then the last block combines them (fixed order)
        double b1 = w1[lane], b2 = w2[lane];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            b1 += __shfl_xor_sync(0xffffffffu, b1, off);
            b2 += __shfl_xor_sync(0xffffffffu, b2, off);
        }
        if (lane == 0) {
            block_sums[2 * blockIdx.x] = b1;
            block_sums[2 * blockIdx.x + 1] = b2;
        }
    }
    if (!done_counter || !with_adv) return;
    __shared__ bool last;
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(done_counter, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double c1 = 0.0, c2 = 0.0;
    for (int k = threadIdx.x; k < static_cast<int>(gridDim.x); k += 1024) {
        c1 += __ldcg(block_sums + 2 * k);
        c2 += __ldcg(block_sums + 2 * k + 1);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        c1 += __shfl_xor_sync(0xffffffffu, c1, off);
        c2 += __shfl_xor_sync(0xffffffffu, c2, off);
    }
    __syncthreads();
    if (lane == 0) {
        w1[w] = c1;
        w2[w] = c2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double t1 = 0.0, t2 = 0.0;
        for (int k = 0; k < 32; ++k) {
            t1 += w1[k];
            t2 += w2[k];
        }
        const double n = static_cast<double>(32 * R);
        const double mean = t1 / n;
        const double var = t2 / n - mean * mean;
        stats[0] = mean;
        stats[1] = sqrt(var > 0.0 ? var : 0.0);
        *done_counter = 0;
    }
}

// ---- MAPPO compact critic (fast numerics, n > 4; programs.cpp:390-402): the critic's layer 0
// over [joint(t,e) | onehot(a)] is P[t,e] = joint . W_J (a cuBLAS TF32 GEMM, once per env)
// plus the row W[J+a]; its gradients come back from the input-gradient stage of k_learn.
template <int ACT>
__global__ void __launch_bounds__(256) k_mappo_h0(const float* __restrict__ P, const float* __restrict__ W0,
                                                  const float* __restrict__ b0, int64_t blocks, int64_t E, int n, int J,
                                                  int H, float* __restrict__ h0) {
    // thread = (row, 4 columns): float4 traffic, 32-bit index math once per row (the row count
    // blocks * n * E and H are far below 2^31)
    const uint32_t H4 = static_cast<uint32_t>(H) / 4, nE = static_cast<uint32_t>(n * E), E32 = static_cast<uint32_t>(E);
    const uint32_t total = static_cast<uint32_t>(blocks) * nE * H4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t c4 = i % H4, row = i / H4, blk = row / nE, rem = row % nE, a = rem / E32, e = rem % E32;
        const float4 p = reinterpret_cast<const float4*>(P + (static_cast<int64_t>(blk) * E + e) * H)[c4];
        // W0 / b0 live inside the flat parameter vector: not 16-byte aligned in general
        const float* w = W0 + static_cast<int64_t>(J + a) * H + 4 * c4;
        const float* b = b0 + 4 * c4;
        float z[4] = {p.x + w[0] + b[0], p.y + w[1] + b[1], p.z + w[2] + b[2], p.w + w[3] + b[3]};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (ACT == 0) asm("tanh.approx.f32 %0, %1;" : "=f"(z[j]) : "f"(z[j]));
            if (ACT == 1) z[j] = fmaxf(z[j], 0.0f);
        }
        reinterpret_cast<float4*>(h0)[i] = make_float4(z[0], z[1], z[2], z[3]);
    }
}

// S[t,e] = sum_a dz0[t,a,e] (the joint rows' gradient, fixed agent order); thread = (t, e, 4 columns)
__global__ void __launch_bounds__(256) k_mappo_sum_agents(const float* __restrict__ dz0, int64_t T, int64_t E, int n,
                                                          int H, float* S) {
    const uint32_t H4 = static_cast<uint32_t>(H) / 4, E32 = static_cast<uint32_t>(E);
    const uint32_t total = static_cast<uint32_t>(T * E) * H4;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const uint32_t c4 = i % H4, te = i / H4, t = te / E32, e = te % E32;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int a = 0; a < n; ++a) {
            const float4 v = reinterpret_cast<const float4*>(dz0 + ((static_cast<int64_t>(t) * n + a) * E + e) * H)[c4];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
        reinterpret_cast<float4*>(S)[i] = acc;
    }
}

// dW_onehot[a][c] = sum_{t,e} dz0[t,a,e][c], in two fixed-order passes: block (t, a) sums its
// E rows (16 row phases x 16 float4 column chunks; the phases combined in order) into
// part[t][a][c], then the T partials are added in order
__global__ void __launch_bounds__(256) k_mappo_onehot_part(const float* __restrict__ dz0, int64_t E, int n, int H,
                                                           float* part) {
    __shared__ float4 ws[16][16];
    const int ch = threadIdx.x & 15, ph = threadIdx.x >> 4;
    const int64_t t = blockIdx.x;
    const int a = blockIdx.y;
    const int H4 = H / 4;
    const float* base = dz0 + ((t * n + a) * E) * H;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ch < H4) {
#pragma unroll 4
        for (int64_t e = ph; e < E; e += 16) {
            const float4 v = reinterpret_cast<const float4*>(base + e * H)[ch];
            acc.x += v.x;
            acc.y += v.y;
            acc.z += v.z;
            acc.w += v.w;
        }
    }
    ws[ph][ch] = acc;
    __syncthreads();
    if (threadIdx.x < H) {
        const int c = threadIdx.x;
        float tsum = 0.0f;
        for (int k = 0; k < 16; ++k) tsum += reinterpret_cast<const float*>(&ws[k][c >> 2])[c & 3];
        part[(t * n + a) * H + c] = tsum;
    }
}

__global__ void k_mappo_onehot_sum(const float* __restrict__ part, int64_t T, int n, int H, float* gWoh) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (a, c)
    if (i >= n * H) return;
    const int a = i / H, c = i % H;
    float s = 0.0f;
    for (int64_t t = 0; t < T; ++t) s += part[(t * n + a) * H + c];
    gWoh[a * H + c] = s;
}

// db0[c] = sum_a dW_onehot[a][c] (every row has exactly one agent)
__global__ void k_mappo_bias_grad(const float* __restrict__ gWoh, int n, int H, float* gb0) {
    const int c = threadIdx.x;
    if (c >= H) return;
    float s = 0.0f;
    for (int a = 0; a < n; ++a) s += gWoh[a * H + c];
    gb0[c] = s;
}

}  // namespace

void mappo_fast_h0(cudaStream_t s, const float* P, const float* W0, const float* b0, int64_t blocks, int64_t E, int n,
                   int J, int H, int act, float* h0) {
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>(8192, (blocks * n * E * H + 255) / 256));
    if (act == 0)
        k_mappo_h0<0><<<nb, 256, 0, s>>>(P, W0, b0, blocks, E, n, J, H, h0);
    else
        k_mappo_h0<1><<<nb, 256, 0, s>>>(P, W0, b0, blocks, E, n, J, H, h0);
}

void mappo_fast_layer0_grads(cudaStream_t s, const float* dz0, int64_t T, int64_t E, int n, int H, float* S,
                             float* part, float* gWoh, float* gb0) {
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>(8192, (T * E * H + 255) / 256));
    k_mappo_sum_agents<<<nb, 256, 0, s>>>(dz0, T, E, n, H, S);
    k_mappo_onehot_part<<<dim3(static_cast<unsigned>(T), n), 256, 0, s>>>(dz0, E, n, H, part);
    k_mappo_onehot_sum<<<(n * H + 255) / 256, 256, 0, s>>>(part, T, n, H, gWoh);
    k_mappo_bias_grad<<<1, 64, 0, s>>>(gWoh, n, H, gb0);
}

namespace {

// Per-replica advantage statistics (R units folded into one engine, each normalising over its
// own T*E_r rows like its own interpreter, rl.cpp:97-107): one CTA per replica, fixed order.
__global__ void __launch_bounds__(256) k_rep_adv_stats(const float* __restrict__ adv, int64_t T, int64_t E,
                                                       const int64_t* __restrict__ rep_off,
                                                       const int64_t* __restrict__ rep_n, double* stats) {
    __shared__ double s1[256], s2[256];
    const int r = blockIdx.x;
    const int64_t off = rep_off[r], er = rep_n[r], n = T * er;
    double a1 = 0.0, a2 = 0.0;
    for (int64_t i = threadIdx.x; i < n; i += 256) {
        const double x = adv[(i / er) * E + off + i % er];
        a1 += x;
        a2 += x * x;
    }
    s1[threadIdx.x] = a1;
    s2[threadIdx.x] = a2;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            s1[threadIdx.x] += s1[threadIdx.x + o];
            s2[threadIdx.x] += s2[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double mean = s1[0] / static_cast<double>(n);
        const double var = s2[0] / static_cast<double>(n) - mean * mean;
        stats[2 * r] = mean;
        stats[2 * r + 1] = sqrt(var > 0.0 ? var : 0.0);
    }
}

// Parallel episode reward sum (fast numerics): block tree sums in double, fixed block order.
__global__ void __launch_bounds__(256) k_block_sum(const double* __restrict__ x, int64_t n, double* block_out) {
    __shared__ double s[256];
    double a = 0.0;
    for (int64_t i = blockIdx.x * 256 + threadIdx.x; i < n; i += static_cast<int64_t>(gridDim.x) * 256) a += x[i];
    s[threadIdx.x] = a;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
        if (threadIdx.x < off) s[threadIdx.x] += s[threadIdx.x + off];
        __syncthreads();
    }
    if (threadIdx.x == 0) block_out[blockIdx.x] = s[0];
}

__global__ void k_sum_blocks(const double* __restrict__ b, int n, double* out) {
    if (threadIdx.x != 0) return;
    double a = 0.0;
    for (int i = 0; i < n; ++i) a += b[i];
    *out = a;
}

}  // namespace

// ------------------------------------------------------------------------------ launchers
size_t fast_wimg_bytes(const FastNet& n) { return carve(n).x; }
size_t fast_hsave_bytes(const FastNet& n) { return carve(n).hbytes; }

void fast_build_wimg(cudaStream_t s, const float* params, const FastNet& n0, __nv_bfloat16* img0, const FastNet& n1,
                     __nv_bfloat16* img1) {
    k_build_wimg<<<dim3(64, 2), 256, 0, s>>>(params, n0, img0, n1, img1);
}


void fast_reduce_partials(cudaStream_t s, const float* part_p, const float* part_c, int np, int nc, int64_t Pp,
                          int64_t Pc, float* grads, int64_t c_off) {
    k_reduce_partials<<<static_cast<unsigned>((Pp + Pc + 31) / 32), 256, 0, s>>>(part_p, part_c, np, nc, Pp, Pc,
                                                                                 c_off, grads);
}

void fast_reduce_adam(cudaStream_t s, const FastUpdateArgs& a, bool pdl) {
    const int64_t padded = (a.Pp + 3) / 4 * 4 + (a.Pc + 3) / 4 * 4;
    const int nchunks = static_cast<int>((padded + 127) / 128);
    const unsigned grid = static_cast<unsigned>(std::min(nchunks, 148 * 8));
    if (!pdl) {
        k_reduce_adam<false><<<grid, 256, 0, s>>>(a, nchunks);
        return;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    FLW_CUDA(cudaLaunchKernelEx(&cfg, k_reduce_adam<true>, a, nchunks));
}

void fast_reduce_loss(cudaStream_t s, const float* loss_parts, int np, int nc, double entropy_coef, float* loss) {
    k_reduce_loss<<<1, 32, 0, s>>>(loss_parts, np, nc, entropy_coef, loss);
}

void fast_gae(cudaStream_t s, const float* rew, const float* values, const float* done_f, const float* last_value,
              int64_t TR, int64_t R, double gamma, double lam, float* adv, float* ret, bool with_adv,
              double* block_sums, double* stats, unsigned* done_counter, bool pdl) {
    // T = 32 with few streams (the episode: latency-bound): warp-shuffle reverse scan, lane = step.
    // Many streams (bandwidth-bound sweeps): the chunked thread-per-stream recurrence, which needs
    // no shuffles (the scan's 40 shuffles per stream would cap it at ~20% of HBM bandwidth).
    // T = 32 and up to 65536 streams (the C2 / C3 / C5 episodes): the warp-shuffle scan, one
    // 32-stream tile per block (latency regime). Many streams: the thread-per-stream recurrence
    // streams HBM faster (2^26 rows: 5.1 vs 1.8 TB/s, bench.py hbm_kernels).
    if (TR == 32 * R && done_counter && R <= 65536) {
        const int nb32 = static_cast<int>(std::min<int64_t>((R + 31) / 32, 2 * 148));
        if (!pdl) {
            k_gae_scan32<<<nb32, 1024, 0, s>>>(rew, values, done_f, last_value, R, gamma, lam, adv, ret, with_adv,
                                               block_sums, stats, done_counter, false);
            return;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(nb32));
        cfg.blockDim = dim3(1024);
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        FLW_CUDA(cudaLaunchKernelEx(&cfg, k_gae_scan32, rew, values, done_f, last_value, R, gamma, lam, adv, ret,
                                    with_adv, block_sums, stats, done_counter, true));
        return;
    }
    const int nb = static_cast<int>((R + 255) / 256);
    // few streams: latency-bound, every step's loads issued at once; many streams (scaled
    // sweeps): occupancy-bound, 8-step chunks at 4 blocks per SM
    if (R <= 65536)
        k_fast_gae<32, 1><<<nb, 256, 0, s>>>(rew, values, done_f, last_value, TR / R, R, gamma, lam, adv, ret,
                                             with_adv, block_sums, stats, done_counter);
    else
        k_fast_gae<8, 4><<<nb, 256, 0, s>>>(rew, values, done_f, last_value, TR / R, R, gamma, lam, adv, ret,
                                            with_adv, block_sums, stats, done_counter);
    if (with_adv && !done_counter) k_adv_stats<<<1, 256, 0, s>>>(block_sums, nb, TR, stats);
}

void fast_gae_scan32(cudaStream_t s, const float* rew, const float* values, const float* done_f,
                     const float* last_value, int64_t R, double gamma, double lam, float* adv, float* ret,
                     bool with_adv, double* block_sums, double* stats, unsigned* done_counter) {
    const int nb32 = static_cast<int>(std::min<int64_t>((R + 31) / 32, 2 * 148));
    k_gae_scan32<<<nb32, 1024, 0, s>>>(rew, values, done_f, last_value, R, gamma, lam, adv, ret, with_adv,
                                       block_sums, stats, done_counter, false);
}

void fast_rep_adv_stats(cudaStream_t s, const float* adv, int64_t T, int64_t E, const int64_t* rep_off,
                        const int64_t* rep_n, int R, double* stats) {
    k_rep_adv_stats<<<R, 256, 0, s>>>(adv, T, E, rep_off, rep_n, stats);
}

void fast_sum(cudaStream_t s, const double* x, int64_t n, double* scratch, double* out) {
    const int nb = static_cast<int>(std::min<int64_t>(148, (n + 255) / 256));
    k_block_sum<<<nb, 256, 0, s>>>(x, n, scratch);
    k_sum_blocks<<<1, 32, 0, s>>>(scratch, nb, out);
}

}  // namespace flw
