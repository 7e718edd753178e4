// Exact-numerics kernels: CUDA-core FP64 accumulation that reproduces the reference
// interpreter's arithmetic bit-for-bit (every tensor op rounds its double result to f32,
// core/tensor.hpp:42-79; reductions run left-to-right from 0.0, compute/ops.hpp:13-14).
//
//   * Dot products use fma(a, b, acc) on f32-valued operands: the f32 x f32 product is exact in
//     double, so fma == acc + a*b with the reference's single rounding, in the same k order.
//   * Every other double expression uses explicit __d*_rn intrinsics (no FMA contraction).
//   * Reductions whose result must match a sequential left-to-right sum (dW/db over all T*E
//     rows, advantage mean/variance, reward and loss sums) run as one chain per output.
// Transcendentals (exp/log/tanh) come from CUDA's libdevice rather than glibc; both are within
// an ulp of the true value and the result is immediately rounded to f32, so they agree except
// on rare f32 rounding ties (tests count those).
#include <cmath>

#include "engine.hpp"
#include "kernels.cuh"

namespace flw {

namespace {

// std::max / std::min value semantics (a < b ? b : a), (b < a ? b : a)
__device__ __forceinline__ double dmax(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }

// --------------------------------------------------------------------------------- reset
// begin (the episode graph): also k_begin_episode's work - the episode is ctx->next_episode, and
// the last block to finish stores it in ctx->episode and advances ctx->next_episode (every block
// has read it by then; begin re-armed to 0)
__global__ void k_reset(DeviceCtx* __restrict__ ctx, EnvParams env, double* est, uint8_t* done,
                        int32_t* stepc, float* obs0, int64_t E, int64_t env_lo, int S, uint64_t seed,
                        unsigned* begin) {
    const int64_t ep = begin ? ctx->next_episode : ctx->episode;
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e < E) {
        // env_seed = key(seed, kEnvStream, env_lo + e, episode)  (interp.cpp:214-215)
        const uint64_t es = rng_key(seed, kEnvStream, static_cast<uint64_t>(env_lo + e), static_cast<uint64_t>(ep));
        env_reset_dev(env, es, est, E, e);
        done[e] = 0;
        stepc[e] = 0;
        for (int j = 0; j < S; ++j) obs0[e * S + j] = static_cast<float>(env_obs1(env, est, E, e, j));
    }
    if (begin) {
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(begin, 1u) == gridDim.x - 1) {
            ctx->episode = ep;
            ctx->next_episode = ep + 1;
            *begin = 0u;
        }
    }
}

// ------------------------------------------------------------------------ dense layers
// 32x32 output tile per CTA (256 threads = 8 warps; lane = column, warp = row group of 4).
// Operands are staged in shared memory as doubles; the k loop never touches padding so the
// accumulation sequence is exactly acc = ((0 + x0*w0) + x1*w1) + ... (ops.cpp:98-104).
template <int ACT>
__global__ void __launch_bounds__(256) k_fwd(const float* __restrict__ in, const float* __restrict__ W,
                                             const float* __restrict__ b, float* __restrict__ out, int64_t M,
                                             int K, int N) {
    __shared__ double As[32][33];
    __shared__ double Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int c0 = blockIdx.y * 32;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int rr = ty + 8 * q;
            int64_t row = r0 + rr;
            int kk = k0 + tx;
            As[rr][tx] = (row < M && kk < K) ? static_cast<double>(in[row * K + kk]) : 0.0;
            int kr = ty + 8 * q;
            int kg = k0 + kr, cc = c0 + tx;
            Bs[kr][tx] = (kg < K && cc < N) ? static_cast<double>(W[static_cast<int64_t>(kg) * N + cc]) : 0.0;
        }
        __syncthreads();
        const int kmax = min(32, K - k0);
        for (int k = 0; k < kmax; ++k) {
            double bv = Bs[k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][k], bv, acc[q]);
        }
        __syncthreads();
    }
    const int col = c0 + tx;
    if (col >= N) return;
    const double bias = static_cast<double>(b[col]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int64_t row = r0 + ty + 8 * q;
        if (row >= M) continue;
        double z = f32r(acc[q]);                 // MatMul node output
        double za = f32r(__dadd_rn(z, bias));    // Add node output
        double h = za;
        if (ACT == kTanh) h = f32r(tanh(za));    // ops::tanh
        if (ACT == kRelu) h = za > 0 ? za : 0.0; // ops::relu
        out[row * N + col] = static_cast<float>(h);
    }
}

// dZ_{l-1} = act'(dH) with dH = dZ_l . W_l^T (matmul_grad_lhs, ops.cpp:213-226) and
// tanh_grad dy*(1-y*y) (ops.cpp:242-246) / relu_grad (ops.cpp:248-252).
template <int ACT>
__global__ void __launch_bounds__(256) k_dh(const float* __restrict__ dz, const float* __restrict__ W,
                                            const float* __restrict__ hprev, float* __restrict__ dzprev, int64_t M,
                                            int K, int N) {
    __shared__ double As[32][33];
    __shared__ double Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int c0 = blockIdx.y * 32;  // over K (the previous layer's width)
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j0 = 0; j0 < N; j0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int rr = ty + 8 * q;
            int64_t row = r0 + rr;
            int jj = j0 + tx;
            As[rr][tx] = (row < M && jj < N) ? static_cast<double>(dz[row * N + jj]) : 0.0;
            int jr = ty + 8 * q;
            int jg = j0 + jr, cc = c0 + tx;
            Bs[jr][tx] = (jg < N && cc < K) ? static_cast<double>(W[static_cast<int64_t>(cc) * N + jg]) : 0.0;
        }
        __syncthreads();
        const int jmax = min(32, N - j0);
        for (int j = 0; j < jmax; ++j) {
            double bv = Bs[j][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][j], bv, acc[q]);
        }
        __syncthreads();
    }
    const int col = c0 + tx;
    if (col >= K) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int64_t row = r0 + ty + 8 * q;
        if (row >= M) continue;
        double d = f32r(acc[q]);
        double y = static_cast<double>(hprev[row * K + col]);
        double g = ACT == kTanh ? f32r(__dmul_rn(d, __dsub_rn(1.0, __dmul_rn(y, y)))) : (y > 0 ? d : 0.0);
        dzprev[row * K + col] = static_cast<float>(g);
    }
}

// ------------------------------------------------------------------------- rollout step
// PolicyApply (interp.cpp:175-203: softmax ops.cpp:108-122, inverse-CDF sample on
// u = U(key(seed, act, ep, step, global_row)), logp = log(max(p, 1e-30))) fused with EnvStep
// (interp.cpp:227-262: absorbing after done, reward 0, done 1) and the trajectory write
// (BufferInsert row block; the next obs lands in the next step's input block directly).
constexpr int kMaxA = 16;

__global__ void k_rollout(const DeviceCtx* __restrict__ ctx, RolloutArgs a) {
    int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= a.E) return;
    const int A = a.A;
    const float* lg = a.logits + e * A;
    double l[kMaxA], p[kMaxA];
    double mx = static_cast<double>(lg[0]);
    for (int c = 0; c < A; ++c) {
        l[c] = static_cast<double>(lg[c]);
        mx = dmax(mx, l[c]);
    }
    double denom = 0.0;
    for (int c = 0; c < A; ++c) denom = __dadd_rn(denom, exp(__dsub_rn(l[c], mx)));
    for (int c = 0; c < A; ++c) p[c] = f32r(__ddiv_rn(exp(__dsub_rn(l[c], mx)), denom));
    double u = rng_uniform(rng_key(a.seed, kActionStream, static_cast<uint64_t>(ctx->episode),
                                   static_cast<uint64_t>(a.step), static_cast<uint64_t>(a.env_lo + e)));
    double cum = 0.0;
    int chosen = A - 1;
    for (int c = 0; c < A; ++c) {
        cum = __dadd_rn(cum, p[c]);
        if (u < cum) {
            chosen = c;
            break;
        }
    }
    a.actions[e] = chosen;
    a.logp[e] = static_cast<float>(log(dmax(p[chosen], 1e-30)));
    if (a.done[e]) {
        a.reward[e] = 0.0f;
        a.reward_d[e] = 0.0;
        a.done_f[e] = 1.0f;
    } else {
        double r;
        int32_t sc = a.stepc[e];
        bool d = env_step1(a.env, a.est, a.E, e, chosen, sc, &r);
        a.stepc[e] = sc + 1;
        a.done[e] = d ? 1 : 0;
        a.reward[e] = static_cast<float>(r);
        a.reward_d[e] = r;
        a.done_f[e] = d ? 1.0f : 0.0f;
    }
    for (int j = 0; j < a.S; ++j) a.next_obs[e * a.S + j] = static_cast<float>(env_obs1(a.env, a.est, a.E, e, j));
}

// --------------------------------------------------------------------- sequential sums
// A left-to-right double sum has to be ONE dependent chain. The block stages the stream through
// double-buffered shared memory (all 256 threads load chunk c+1 while thread 0 adds chunk c), so
// the chain runs at DADD latency instead of global-load latency.
constexpr int kSeqThreads = 256;
constexpr int kSeqChunk = 2048;

// mode 0: sum x; mode 1: sum (x - center)^2, each term individually rounded.
__device__ double seq_chain(const double* __restrict__ x, int64_t n, int mode, double center, double (*buf)[kSeqChunk]) {
    const int t = threadIdx.x;
    auto load = [&](int64_t c, int slot) {
        const int64_t base = c * kSeqChunk;
        for (int i = t; i < kSeqChunk; i += kSeqThreads) buf[slot][i] = base + i < n ? x[base + i] : 0.0;
    };
    const int64_t nchunks = (n + kSeqChunk - 1) / kSeqChunk;
    double acc = 0.0;
    load(0, 0);
    __syncthreads();
    for (int64_t c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) load(c + 1, (c + 1) & 1);
        if (t == 0) {
            const double* b = buf[c & 1];
            const int m = static_cast<int>(min(static_cast<int64_t>(kSeqChunk), n - c * kSeqChunk));
            if (mode == 0) {
                for (int i = 0; i < m; ++i) acc = __dadd_rn(acc, b[i]);
            } else {
                for (int i = 0; i < m; ++i) {
                    double d = __dsub_rn(b[i], center);
                    acc = __dadd_rn(acc, __dmul_rn(d, d));
                }
            }
        }
        __syncthreads();
    }
    return acc;
}

__global__ void __launch_bounds__(kSeqThreads) k_seq_sum(const double* __restrict__ x, int64_t n, double* out) {
    __shared__ double buf[2][kSeqChunk];
    double acc = seq_chain(x, n, 0, 0.0, buf);
    if (threadIdx.x == 0) *out = acc;
}

// -------------------------------------------------------------------------- GAE/returns
// gae_streams / discounted_return_streams (rl.cpp:14-95): one thread per stream s owning the
// t-major rows t*R + s; coalesced across the warp at every t.
__global__ void k_gae(const float* __restrict__ rew, const float* __restrict__ values, const float* __restrict__ done_f,
                      const float* __restrict__ last_value, int64_t T, int64_t R, double gamma, double lam,
                      double* adv_d, float* ret, bool with_adv) {
    int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (s >= R) return;
    const double gl = __dmul_rn(gamma, lam);
    const double lv = static_cast<double>(last_value[s]);
    double acc = 0.0, running = lv;
    for (int64_t t = T - 1; t >= 0; --t) {
        int64_t i = t * R + s;
        bool done = done_f[i] > 0.5f;
        double r = static_cast<double>(rew[i]);
        if (with_adv) {
            double next_v = t + 1 < T ? static_cast<double>(values[i + R]) : lv;
            if (done) {
                next_v = 0.0;
                acc = 0.0;
            }
            double delta = __dsub_rn(__dadd_rn(r, __dmul_rn(gamma, next_v)), static_cast<double>(values[i]));
            acc = __dadd_rn(delta, __dmul_rn(gl, acc));
            adv_d[i] = acc;
        }
        if (done) running = 0.0;
        running = __dadd_rn(r, __dmul_rn(gamma, running));
        ret[i] = static_cast<float>(running);
    }
}

// normalize_advantages (rl.cpp:97-107): sequential mean, then sequential variance.
__global__ void __launch_bounds__(kSeqThreads) k_norm_stats(const double* __restrict__ a, int64_t n, double* stats) {
    __shared__ double buf[2][kSeqChunk];
    __shared__ double mean_s;
    double s = seq_chain(a, n, 0, 0.0, buf);
    if (threadIdx.x == 0) mean_s = __ddiv_rn(s, static_cast<double>(n));
    __syncthreads();
    const double mean = mean_s;
    double var = seq_chain(a, n, 1, mean, buf);
    if (threadIdx.x == 0) {
        stats[0] = mean;
        stats[1] = __dsqrt_rn(__ddiv_rn(var, static_cast<double>(n)));
    }
}

__global__ void k_norm_apply(const double* __restrict__ a, int64_t n, const double* __restrict__ stats, bool normalize,
                             float* out) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double v = a[i];
    if (normalize) {
        double sd = stats[1];
        if (!(sd < 1e-8)) v = __ddiv_rn(__dsub_rn(v, stats[0]), __dadd_rn(sd, 1e-8));
    }
    out[i] = static_cast<float>(v);
}

// ------------------------------------------------------------------------------- losses
// ppo_loss_core (rl.cpp:137-172) / a3c_loss_core (rl.cpp:174-202) per row, with row_dist
// (rl.cpp:117-133). Per-row loss terms go to `terms` for the sequential loss reduction.
__global__ void k_loss_rows(int algo, const float* __restrict__ logits, const float* __restrict__ values,
                            const int32_t* __restrict__ actions, const float* __restrict__ logp_old,
                            const float* __restrict__ adv, const float* __restrict__ ret, int64_t n, int A,
                            double clip_eps, double vc, double ec, float* dlogits, float* dvalues, double* terms) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    double l[kMaxA], p[kMaxA], lp[kMaxA];
    double mx = static_cast<double>(logits[i * A]);
    for (int j = 0; j < A; ++j) {
        l[j] = static_cast<double>(logits[i * A + j]);
        mx = dmax(mx, l[j]);
    }
    double denom = 0.0;
    for (int j = 0; j < A; ++j) denom = __dadd_rn(denom, exp(__dsub_rn(l[j], mx)));
    double log_denom = log(denom);
    double H = 0.0;
    for (int j = 0; j < A; ++j) {
        lp[j] = __dsub_rn(__dsub_rn(l[j], mx), log_denom);
        p[j] = exp(lp[j]);
        H = __dsub_rn(H, __dmul_rn(p[j], lp[j]));
    }
    const double inv_n = __ddiv_rn(1.0, static_cast<double>(n));
    const int a = actions[i];
    const double v = static_cast<double>(values[i]), R = static_cast<double>(ret[i]);
    double coef, pl;
    if (algo == 0) {  // PPO clipped surrogate
        double A_ = static_cast<double>(adv[i]);
        double ratio = exp(__dsub_rn(lp[a], static_cast<double>(logp_old[i])));
        double clipped = dmin(dmax(ratio, __dsub_rn(1.0, clip_eps)), __dadd_rn(1.0, clip_eps));
        double s1 = __dmul_rn(ratio, A_), s2 = __dmul_rn(clipped, A_);
        pl = __dmul_rn(dmin(s1, s2), inv_n);
        coef = s1 <= s2 ? __dmul_rn(__dmul_rn(-inv_n, ratio), A_) : 0.0;
    } else {  // A3C: advantage R - V held constant
        double A_ = __dsub_rn(R, v);
        pl = __dmul_rn(__dmul_rn(lp[a], A_), inv_n);
        coef = __dmul_rn(-inv_n, A_);
    }
    double verr = __dsub_rn(v, R);
    double vl = __dmul_rn(__dmul_rn(__dmul_rn(vc, verr), verr), inv_n);
    double dv = __dmul_rn(__dmul_rn(__dmul_rn(2.0, vc), verr), inv_n);
    double en = __dmul_rn(H, inv_n);
    const double eci = __dmul_rn(ec, inv_n);
    for (int j = 0; j < A; ++j) {
        double g = __dmul_rn(coef, __dsub_rn(j == a ? 1.0 : 0.0, p[j]));
        g = __dadd_rn(g, __dmul_rn(__dmul_rn(eci, p[j]), __dadd_rn(lp[j], H)));
        dlogits[i * A + j] = static_cast<float>(g);
    }
    dvalues[i] = static_cast<float>(dv);  // backward_flat: dv.set(g * dvalues[i]) with g = 1
    terms[i] = pl;
    terms[n + i] = vl;
    terms[2 * n + i] = en;
}

__global__ void k_loss_reduce(const double* __restrict__ terms, int64_t n, double ec, float* loss) {
    double pl = 0.0, vl = 0.0, en = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        pl = __dsub_rn(pl, terms[i]);
        vl = __dadd_rn(vl, terms[n + i]);
        en = __dadd_rn(en, terms[2 * n + i]);
    }
    *loss = static_cast<float>(__dsub_rn(__dadd_rn(pl, vl), __dmul_rn(ec, en)));
}

// ------------------------------------------------------------------------------ dW / db
// matmul_grad_rhs (ops.cpp:228-240) and reduce_to_shape (ops.cpp:267-277): one sequential
// chain over ALL rows per weight (bit-exactness forbids split-K). Tile = 32 t x 32 j; a thread
// owns 4 t's x 1 j. The bias is the extra row t == K with h == 1 (1*dz is exact). The next
// 128-row chunk is prefetched into registers while the current one is consumed from smem, so
// the chains run at DFMA latency rather than global-load latency.
constexpr int kDwRows = 128;
constexpr int kDwPer = kDwRows / 8;  // rows per thread per chunk (8 warps)

__global__ void __launch_bounds__(256) k_dw(const DwTile* __restrict__ tiles) {
    extern __shared__ double dw_smem[];
    double(*Hs)[kDwRows][33] = reinterpret_cast<double(*)[kDwRows][33]>(dw_smem);
    double(*Ds)[kDwRows][33] = reinterpret_cast<double(*)[kDwRows][33]>(dw_smem + 2 * kDwRows * 33);
    const DwTile tl = tiles[blockIdx.x];
    const int64_t M = tl.rows;
    const int tx = threadIdx.x & 31, tg = threadIdx.x >> 5;
    const int K = tl.K, N = tl.N;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    float hreg[kDwPer], dreg[kDwPer];
    auto fetch = [&](int64_t i0) {
#pragma unroll
        for (int q = 0; q < kDwPer; ++q) {
            int rr = tg + 8 * q;
            int64_t row = i0 + rr;
            int t = tl.t0 + tx, j = tl.j0 + tx;
            if (tl.cn > 0 && row < M && t < K) {  // compact MAPPO critic input [joint | one-hot]
                const int64_t per = static_cast<int64_t>(tl.cn) * tl.cE;
                const int64_t tb = row / per, rem = row % per, a = rem / tl.cE, e = rem % tl.cE;
                hreg[q] = t < tl.cJ ? tl.H[(tb * tl.cE + e) * tl.cJ + t] : (t - tl.cJ == a ? 1.0f : 0.0f);
            } else {
                hreg[q] = row < M ? (t < K ? tl.H[row * K + t] : (t == K ? 1.0f : 0.0f)) : 0.0f;
            }
            dreg[q] = (row < M && j < N) ? tl.DZ[row * N + j] : 0.0f;
        }
    };
    auto stash = [&](int buf) {
#pragma unroll
        for (int q = 0; q < kDwPer; ++q) {
            Hs[buf][tg + 8 * q][tx] = static_cast<double>(hreg[q]);
            Ds[buf][tg + 8 * q][tx] = static_cast<double>(dreg[q]);
        }
    };
    fetch(0);
    stash(0);
    __syncthreads();
    int buf = 0;
    for (int64_t i0 = 0; i0 < M; i0 += kDwRows) {
        const bool more = i0 + kDwRows < M;
        if (more) fetch(i0 + kDwRows);
        const int rows = M - i0 < kDwRows ? static_cast<int>(M - i0) : kDwRows;
        for (int r = 0; r < rows; ++r) {
            double d = Ds[buf][r][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(Hs[buf][r][tg * 4 + q], d, acc[q]);
        }
        if (more) stash(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    const int j = tl.j0 + tx;
    if (j >= N) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int t = tl.t0 + tg * 4 + q;
        if (t < K)
            tl.gW[static_cast<int64_t>(t) * N + j] = static_cast<float>(acc[q]);
        else if (t == K)
            tl.gB[j] = static_cast<float>(acc[q]);
    }
}

// ------------------------------------------------------------------------ GradSync + Adam
// GradSync mean (local_run.cpp:408-411): sum over units in unit-id order from 0.0, then / k.
__global__ void k_grad_mean(const float* __restrict__ g, int k, int64_t P, double* mean) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    double acc = 0.0;
    for (int r = 0; r < k; ++r) acc = __dadd_rn(acc, static_cast<double>(g[r * P + i]));
    mean[i] = __ddiv_rn(acc, static_cast<double>(k));
}

__global__ void k_begin_episode(DeviceCtx* ctx) { ctx->episode = ctx->next_episode++; }

// The episode's reward sums into slot (runs % slots) of a host-mapped ring (zero-copy: no
// device-to-host copy between two episode graphs); the host reads the slot after the episode's
// completion event.
__global__ void k_publish_rsum(DeviceCtx* ctx, const double* rsum, int n, double* ring, int slots) {
    const uint64_t slot = ctx->runs % static_cast<uint64_t>(slots);
    for (int i = 0; i < n; ++i) ring[slot * n + i] = rsum[i];
    __threadfence_system();
    ctx->runs += 1;
}

__global__ void k_adam_tick(DeviceCtx* ctx, const double2* __restrict__ table, int64_t len) {
    int64_t t = ++ctx->adam_t;
    if (t <= len) {
        ctx->bc1 = table[t - 1].x;
        ctx->bc2 = table[t - 1].y;
    } else {  // beyond the host table: device pow (ulp-level deviation possible)
        ctx->bc1 = 1.0 - pow(0.9, static_cast<double>(t));
        ctx->bc2 = 1.0 - pow(0.999, static_cast<double>(t));
    }
}

// adam_step (mlp.cpp:146-161): double moments, f32 params.
__global__ void k_adam(const DeviceCtx* __restrict__ ctx, float* params, const float* __restrict__ g32,
                       const double* __restrict__ g64, double* m, double* v, int64_t P, double lr, double b1,
                       double b2, double eps, double gscale) {
    int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (i >= P) return;
    const double bc1 = ctx->bc1, bc2 = ctx->bc2;
    double g = g64 ? g64[i] : __dmul_rn(static_cast<double>(g32[i]), gscale);
    double mi = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(__dsub_rn(1.0, b1), g));
    double vi = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, b2), g), g));
    m[i] = mi;
    v[i] = vi;
    double mhat = __ddiv_rn(mi, bc1), vhat = __ddiv_rn(vi, bc2);
    double next = __dsub_rn(static_cast<double>(params[i]),
                            __ddiv_rn(__dmul_rn(lr, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
    params[i] = static_cast<float>(next);
}

inline unsigned blocks_for(int64_t n, int t) { return static_cast<unsigned>((n + t - 1) / t); }

}  // namespace

// ------------------------------------------------------------------------------ launchers
void exact_reset(cudaStream_t s, DeviceCtx* ctx, const EnvParams& env, double* est, uint8_t* done,
                 int32_t* stepc, float* obs0, int64_t E, int64_t env_lo, int S, uint64_t seed, unsigned* begin) {
    k_reset<<<blocks_for(E, 128), 128, 0, s>>>(ctx, env, est, done, stepc, obs0, E, env_lo, S, seed, begin);
}

void exact_layer_fwd(cudaStream_t s, const float* in, const float* W, const float* b, float* out, int64_t M, int K,
                     int N, int act) {
    dim3 grid(blocks_for(M, 32), blocks_for(N, 32));
    if (act == kTanh)
        k_fwd<kTanh><<<grid, 256, 0, s>>>(in, W, b, out, M, K, N);
    else if (act == kRelu)
        k_fwd<kRelu><<<grid, 256, 0, s>>>(in, W, b, out, M, K, N);
    else
        k_fwd<kNone><<<grid, 256, 0, s>>>(in, W, b, out, M, K, N);
}

void exact_layer_dh(cudaStream_t s, const float* dz, const float* W, const float* hprev, float* dzprev, int64_t M,
                    int K, int N, int act) {
    dim3 grid(blocks_for(M, 32), blocks_for(K, 32));
    if (act == kTanh)
        k_dh<kTanh><<<grid, 256, 0, s>>>(dz, W, hprev, dzprev, M, K, N);
    else
        k_dh<kRelu><<<grid, 256, 0, s>>>(dz, W, hprev, dzprev, M, K, N);
}

void exact_rollout(cudaStream_t s, const DeviceCtx* ctx, const RolloutArgs& a) {
    k_rollout<<<blocks_for(a.E, 128), 128, 0, s>>>(ctx, a);
}

void exact_seq_sum(cudaStream_t s, const double* x, int64_t n, double* out) {
    k_seq_sum<<<1, kSeqThreads, 0, s>>>(x, n, out);
}

void exact_gae(cudaStream_t s, const float* rew, const float* values, const float* done_f, const float* last_value,
               int64_t TR, int64_t R, double gamma, double lam, double* adv_d, float* ret, bool with_adv) {
    k_gae<<<blocks_for(R, 128), 128, 0, s>>>(rew, values, done_f, last_value, TR / R, R, gamma, lam, adv_d, ret,
                                             with_adv);
}

void exact_normalize(cudaStream_t s, const double* adv_d, int64_t n, bool normalize, double* stats, float* adv) {
    if (normalize) k_norm_stats<<<1, kSeqThreads, 0, s>>>(adv_d, n, stats);
    k_norm_apply<<<blocks_for(n, 256), 256, 0, s>>>(adv_d, n, stats, normalize, adv);
}

void exact_loss_rows(cudaStream_t s, int algo, const float* logits, const float* values, const int32_t* actions,
                     const float* logp_old, const float* adv, const float* ret, int64_t n, int A, double clip_eps,
                     double value_coef, double entropy_coef, float* dlogits, float* dvalues, double* terms) {
    k_loss_rows<<<blocks_for(n, 128), 128, 0, s>>>(algo, logits, values, actions, logp_old, adv, ret, n, A, clip_eps,
                                                   value_coef, entropy_coef, dlogits, dvalues, terms);
}

void exact_loss_reduce(cudaStream_t s, const double* terms, int64_t n, double entropy_coef, float* loss) {
    k_loss_reduce<<<1, 1, 0, s>>>(terms, n, entropy_coef, loss);
}

template <typename V>
__global__ void k_permute_rows(const V* __restrict__ src, V* __restrict__ dst, int64_t T, int64_t E, int w,
                               ReplicaMap m) {
    const int64_t n = T * E * w;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = i % w, row = i / w, t = row / E, e = row % E;
        const int r = m.rep_of_env[e];
        const int64_t off = m.rep_off[r], er = m.rep_n[r];
        dst[((T * off + t * er) + (e - off)) * w + c] = src[i];
    }
}

void permute_rows_f32(cudaStream_t s, const float* src, float* dst, int64_t T, int64_t E, int w, const ReplicaMap& m) {
    k_permute_rows<float><<<static_cast<unsigned>(std::min<int64_t>(4096, blocks_for(T * E * w, 256))), 256, 0, s>>>(
        src, dst, T, E, w, m);
}
void permute_rows_i32(cudaStream_t s, const int32_t* src, int32_t* dst, int64_t T, int64_t E, const ReplicaMap& m) {
    k_permute_rows<int32_t><<<static_cast<unsigned>(std::min<int64_t>(4096, blocks_for(T * E, 256))), 256, 0, s>>>(
        src, dst, T, E, 1, m);
}
void permute_rows_f64(cudaStream_t s, const double* src, double* dst, int64_t T, int64_t E, const ReplicaMap& m) {
    k_permute_rows<double><<<static_cast<unsigned>(std::min<int64_t>(4096, blocks_for(T * E, 256))), 256, 0, s>>>(
        src, dst, T, E, 1, m);
}

// joint prefix chains: prefix[r][c] = sum_i joint[r][i] * W0[i][c], i ascending from 0.0 (the
// first J terms of the reference's dot over [joint | one-hot]), kept in double.
__global__ void __launch_bounds__(256) k_mappo_prefix(const float* __restrict__ in, const float* __restrict__ W,
                                                      double* __restrict__ out, int64_t M, int K, int N) {
    __shared__ double As[32][33];
    __shared__ double Bs[32][33];
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int64_t r0 = static_cast<int64_t>(blockIdx.x) * 32;
    const int c0 = blockIdx.y * 32;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k0 = 0; k0 < K; k0 += 32) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            int rr = ty + 8 * q;
            int64_t row = r0 + rr;
            int kk = k0 + tx;
            As[rr][tx] = (row < M && kk < K) ? static_cast<double>(in[row * K + kk]) : 0.0;
            int kr = ty + 8 * q;
            int kg = k0 + kr, cc = c0 + tx;
            Bs[kr][tx] = (kg < K && cc < N) ? static_cast<double>(W[static_cast<int64_t>(kg) * N + cc]) : 0.0;
        }
        __syncthreads();
        const int kmax = min(32, K - k0);
        for (int k = 0; k < kmax; ++k) {
            double bv = Bs[k][tx];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = fma(As[ty + 8 * q][k], bv, acc[q]);
        }
        __syncthreads();
    }
    const int col = c0 + tx;
    if (col >= N) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        int64_t row = r0 + ty + 8 * q;
        if (row < M) out[row * N + col] = acc[q];
    }
}

template <int ACT>
__global__ void k_mappo_expand0(const double* __restrict__ prefix, const float* __restrict__ W, const float* __restrict__ b,
                                int64_t blocks, int64_t E, int n, int J, int N, float* out_rows, float* out_last) {
    const int64_t total = blocks * n * E * N;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int c = static_cast<int>(i % N);
        const int64_t row = i / N;  // (blk, a, e) agent-major inside a block
        const int64_t blk = row / (n * E), rem = row % (n * E), a = rem / E, e = rem % E;
        const double acc = __dadd_rn(prefix[(blk * E + e) * N + c], static_cast<double>(W[(J + a) * N + c]));
        double z = f32r(acc);
        double za = f32r(__dadd_rn(z, static_cast<double>(b[c])));
        double h = za;
        if (ACT == kTanh) h = f32r(tanh(za));
        if (ACT == kRelu) h = za > 0 ? za : 0.0;
        float* dst = blk + 1 < blocks ? out_rows + row * N : out_last + rem * N;
        dst[c] = static_cast<float>(h);
    }
}

void exact_mappo_critic0(cudaStream_t s, const float* joint, const float* W0, const float* b0, int64_t blocks,
                         int64_t E, int n, int J, int N, double* prefix, float* out_rows, float* out_last, int act) {
    const int64_t M = blocks * E;
    dim3 g(static_cast<unsigned>((M + 31) / 32), static_cast<unsigned>((N + 31) / 32));
    k_mappo_prefix<<<g, 256, 0, s>>>(joint, W0, prefix, M, J, N);
    const unsigned nb = static_cast<unsigned>(std::min<int64_t>(8192, blocks_for(blocks * n * E * N, 256)));
    if (act == kTanh)
        k_mappo_expand0<kTanh><<<nb, 256, 0, s>>>(prefix, W0, b0, blocks, E, n, J, N, out_rows, out_last);
    else if (act == kRelu)
        k_mappo_expand0<kRelu><<<nb, 256, 0, s>>>(prefix, W0, b0, blocks, E, n, J, N, out_rows, out_last);
    else
        k_mappo_expand0<kNone><<<nb, 256, 0, s>>>(prefix, W0, b0, blocks, E, n, J, N, out_rows, out_last);
}

void exact_dw(cudaStream_t s, const DwTile* tiles, int ntiles) {
    const size_t smem = 4 * kDwRows * 33 * sizeof(double);
    // per-device attribute: set on every launch (cheap, and legal inside stream capture)
    FLW_CUDA(cudaFuncSetAttribute(k_dw, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    if (ntiles > 0) k_dw<<<ntiles, 256, smem, s>>>(tiles);
}

void exact_grad_mean(cudaStream_t s, const float* gathered, int k, int64_t P, double* mean) {
    k_grad_mean<<<blocks_for(P, 256), 256, 0, s>>>(gathered, k, P, mean);
}

void begin_episode(cudaStream_t s, DeviceCtx* ctx) { k_begin_episode<<<1, 1, 0, s>>>(ctx); }

// All parameters in one launch: weights of layer l (woff[l], n[l] elements) Xavier-uniform with
// bound a[l], everything else (biases) zero; optionally the Adam moments zeroed too.
__global__ void k_param_init(XavierTable t, float* params, int64_t P, double* m, double* v, uint64_t seed) {
    for (int64_t j = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; j < P;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float w = 0.0f;
        for (int l = 0; l < t.count; ++l) {
            const int64_t i = j - t.woff[l];
            if (i >= 0 && i < t.n[l]) {
                w = static_cast<float>(rng_uniform_range(rng_key(seed, kParamStream, t.node[l], static_cast<uint64_t>(i)),
                                                         -t.a[l], t.a[l]));
                break;
            }
        }
        params[j] = w;
        if (m) m[j] = 0.0;
        if (v) v[j] = 0.0;
    }
}
void param_init(cudaStream_t s, const XavierTable& t, float* params, int64_t P, double* m, double* v,
                uint64_t seed) {
    if (P > 0) k_param_init<<<static_cast<unsigned>(std::min<int64_t>(blocks_for(P, 256), 148 * 8)), 256, 0, s>>>(
        t, params, P, m, v, seed);
}
void publish_rsum(cudaStream_t s, DeviceCtx* ctx, const double* rsum, int n, double* ring, int slots) {
    k_publish_rsum<<<1, 1, 0, s>>>(ctx, rsum, n, ring, slots);
}

void adam_tick(cudaStream_t s, DeviceCtx* ctx, const double2* bc_table, int64_t table_len) {
    k_adam_tick<<<1, 1, 0, s>>>(ctx, bc_table, table_len);
}

void exact_adam(cudaStream_t s, const DeviceCtx* ctx, float* params, const float* g32, const double* g64, double* m,
                double* v, int64_t P, double lr, double b1, double b2, double eps, double gscale) {
    k_adam<<<blocks_for(P, 256), 256, 0, s>>>(ctx, params, g32, g64, m, v, P, lr, b1, b2, eps, gscale);
}

}  // namespace flw
