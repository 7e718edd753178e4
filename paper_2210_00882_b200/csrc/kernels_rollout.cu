// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 16 envs for
// the episode, 16 threads per env (a "group" = half a warp). Env state lives in registers
// spread over the group, the policy weights are staged in shared memory once, and every step
// runs policy MLP (f32 packed FFMA2, each thread 4 outputs) -> PolicyApply (the reference's
// double-precision softmax / inverse-CDF sampling on the f32 logits, interp.cpp:175-203, the
// per-action exps spread over the group, the order-sensitive sums gathered to the leader) ->
// EnvStep (bit-exact double dynamics; synth17x6 state component q on lane q) -> trajectory
// write, with no HBM round trip of env state or activations between steps.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.hpp"
#include "fast.cuh"

namespace flw {

namespace {

constexpr int kEnvsPerCta = 16;
constexpr int kPerEnv = 16;                       // threads per env: each owns 4 of <= 64 outputs
constexpr int kThreads = kEnvsPerCta * kPerEnv;   // 256 (2 CTAs per SM at the C2 shape)
constexpr int kHStride = 68;   // activation row stride (floats): 16B aligned, spreads banks
constexpr unsigned kFull = 0xffffffffu;

__host__ __device__ inline int pad4(int x) { return (x + 3) & ~3; }

struct RolloutSmem {
    uint32_t w[kMaxLayers], b[kMaxLayers], h[2], total;
};

// W_l stored [pad4(in) x pad4(out)] row-major (zero padded) so the input loop runs in float4 steps.
__host__ __device__ inline RolloutSmem rollout_carve(const FastRolloutArgs& a) {
    RolloutSmem s{};
    uint32_t off = 0;
    for (int l = 0; l < a.L; ++l) {
        s.w[l] = off;
        off += static_cast<uint32_t>(pad4(a.dims[l]) * pad4(a.dims[l + 1]) * 4);
        s.b[l] = off;
        off += static_cast<uint32_t>(pad4(a.dims[l + 1]) * 4);
    }
    s.h[0] = off;
    off += kEnvsPerCta * kHStride * 4;
    s.h[1] = off;
    off += kEnvsPerCta * kHStride * 4;
    s.total = off;
    return s;
}

__device__ __forceinline__ double dmaxd(double a, double b) { return a < b ? b : a; }
__device__ __forceinline__ double gshfl(double v, int src) { return __shfl_sync(kFull, v, src, kPerEnv); }
__device__ __forceinline__ float gshflf(float v, int src) { return __shfl_sync(kFull, v, src, kPerEnv); }
__device__ __forceinline__ int gshfli(int v, int src) { return __shfl_sync(kFull, v, src, kPerEnv); }

template <int ENV>
__global__ void __launch_bounds__(kThreads) k_rollout_episode(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const RolloutSmem S = rollout_carve(a);
    const int t = threadIdx.x, q = t & (kPerEnv - 1), r = t / kPerEnv;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * kEnvsPerCta + r;
    const bool live = e < a.E;
    const int64_t E = a.E;
    const int S_ = a.S, A = a.A;
    // weights: W_l [in x out] row-major, in and out padded to multiples of 4 (zeros)
    for (int l = 0; l < a.L; ++l) {
        const int in = a.dims[l], out = a.dims[l + 1], op = pad4(out), ip = pad4(in);
        float* W = reinterpret_cast<float*>(smem + S.w[l]);
        float* B = reinterpret_cast<float*>(smem + S.b[l]);
        for (int i = t; i < ip * op; i += kThreads) {
            int ii = i / op, o = i % op;
            W[i] = (o < out && ii < in) ? a.params[a.woff[l] + ii * out + o] : 0.0f;
        }
        for (int o = t; o < op; o += kThreads) B[o] = o < out ? a.params[a.boff[l] + o] : 0.0f;
    }
    // zero both activation buffers once: padded input columns must read as 0
    for (int i = t; i < 2 * kEnvsPerCta * kHStride; i += kThreads) reinterpret_cast<float*>(smem + S.h[0])[i] = 0.0f;
    __syncthreads();
    // env state -> registers. gridline: (x, len) on the leader. synth17x6: component q on lane q,
    // component 16 also on lane 0 (s16).
    double sq_own = 0.0, s16 = 0.0, gx = 0.0, glen = 0.0;
    bool done = false;
    int32_t stepc = 0;
    if (live) {
        if (ENV == 0) {
            gx = a.est[e];
            glen = a.est[E + e];
        } else {
            sq_own = a.est[q * E + e];
            if (q == 0) s16 = a.est[16 * E + e];
        }
        done = a.done[e] != 0;
        stepc = a.stepc[e];
    }
    // step-0 policy input: the observation in trajectory block step0
    float* h0 = reinterpret_cast<float*>(smem + S.h[0]);
    for (int j = q; j < S_; j += kPerEnv) h0[r * kHStride + j] = live ? a.states[(a.step0 * E + e) * S_ + j] : 0.0f;
    __syncthreads();
    const uint64_t ep = static_cast<uint64_t>(ctx->episode);

    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
        int cur = 0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], op = pad4(out);
            const float* W = reinterpret_cast<const float*>(smem + S.w[l]);
            const float* B = reinterpret_cast<const float*>(smem + S.b[l]);
            const float* hin = reinterpret_cast<const float*>(smem + S.h[cur]) + r * kHStride;
            float* hout = reinterpret_cast<float*>(smem + S.h[cur ^ 1]) + r * kHStride;
            const bool last = l + 1 == a.L;
            // thread q owns outputs [4q, 4q+4): one float4 of inputs (LDS.128, broadcast to the
            // env's 16 threads) feeds 16 FMAs as packed FFMA2 over two partial sums (even/odd
            // input quads) for instruction-level parallelism
            const int o0 = 4 * q;
            if (o0 < op) {
                float2 lo0 = make_float2(0.f, 0.f), hi0 = lo0, lo1 = lo0, hi1 = lo0;
                const float4* W4 = reinterpret_cast<const float4*>(W) + q;
                const float4* X4 = reinterpret_cast<const float4*>(hin);
                const int op4 = op / 4, ip4 = pad4(in) / 4;
                int i4 = 0;
                for (; i4 + 1 < ip4; i4 += 2) {
                    const float4 x0 = X4[i4], x1 = X4[i4 + 1];
                    const float xs0[4] = {x0.x, x0.y, x0.z, x0.w}, xs1[4] = {x1.x, x1.y, x1.z, x1.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 w0 = W4[(4 * i4 + u) * op4];
                        const float4 w1 = W4[(4 * i4 + 4 + u) * op4];
                        lo0 = __ffma2_rn(make_float2(xs0[u], xs0[u]), make_float2(w0.x, w0.y), lo0);
                        hi0 = __ffma2_rn(make_float2(xs0[u], xs0[u]), make_float2(w0.z, w0.w), hi0);
                        lo1 = __ffma2_rn(make_float2(xs1[u], xs1[u]), make_float2(w1.x, w1.y), lo1);
                        hi1 = __ffma2_rn(make_float2(xs1[u], xs1[u]), make_float2(w1.z, w1.w), hi1);
                    }
                }
                if (i4 < ip4) {
                    const float4 x0 = X4[i4];
                    const float xs0[4] = {x0.x, x0.y, x0.z, x0.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 w0 = W4[(4 * i4 + u) * op4];
                        lo0 = __ffma2_rn(make_float2(xs0[u], xs0[u]), make_float2(w0.x, w0.y), lo0);
                        hi0 = __ffma2_rn(make_float2(xs0[u], xs0[u]), make_float2(w0.z, w0.w), hi0);
                    }
                }
                float v[4] = {(lo0.x + lo1.x) + B[o0], (lo0.y + lo1.y) + B[o0 + 1], (hi0.x + hi1.x) + B[o0 + 2],
                              (hi0.y + hi1.y) + B[o0 + 3]};
                if (!last) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = a.act == 0 ? tanhf(v[j]) : fmaxf(v[j], 0.0f);
                }
                *reinterpret_cast<float4*>(hout + o0) = make_float4(v[0], v[1], v[2], v[3]);
            }
            __syncthreads();
            cur ^= 1;
        }
        const float* logits = reinterpret_cast<const float*>(smem + S.h[cur]) + r * kHStride;
        float* next = reinterpret_cast<float*>(smem + S.h[cur ^ 1]) + r * kHStride;  // next step's layer-0 input
        // ---- PolicyApply over the group: lane c < A owns action c
        double lq = q < A ? static_cast<double>(logits[q]) : -1e300;
        double mx = lq;
#pragma unroll
        for (int off = 8; off > 0; off >>= 1) mx = dmaxd(mx, __shfl_xor_sync(kFull, mx, off, kPerEnv));
        const double eq = q < A ? exp(__dsub_rn(lq, mx)) : 0.0;
        double den = 0.0;  // ordered sum, as ops.cpp:117-118
        for (int c = 0; c < A; ++c) den = __dadd_rn(den, gshfl(eq, c));
        const double pq = q < A ? f32r(__ddiv_rn(eq, den)) : 0.0;
        int chosen = A - 1;
        {
            const double u = rng_uniform(rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step),
                                                 static_cast<uint64_t>(a.env_lo + e)));
            double cum = 0.0;
            bool found = false;
            for (int c = 0; c < A; ++c) {
                cum = __dadd_rn(cum, gshfl(pq, c));
                if (!found && u < cum) {
                    chosen = c;
                    found = true;
                }
            }
        }
        const double pch = gshfl(pq, chosen);
        const int64_t ti = step * E + e;
        if (live && q == 0) {
            a.actions[ti] = chosen;
            a.logp[ti] = static_cast<float>(log(dmaxd(pch, 1e-30)));
        }
        // ---- EnvStep (absorbing after done, interp.cpp:239-245)
        double rew = 0.0;
        bool d = done;
        if (ENV == 0) {
            if (!done) {  // gridline, envs.cpp:38-53 (uniform across the group)
                int64_t len = static_cast<int64_t>(glen), x = static_cast<int64_t>(gx);
                x += chosen == 1 ? 1 : -1;
                if (x < 0) x = 0;
                if (x > len - 1) x = len - 1;
                gx = static_cast<double>(x);
                d = false;
                if (x == len - 1) {
                    rew = 1.0;
                    d = true;
                }
            }
            const float o = static_cast<float>(__ddiv_rn(gx, __dsub_rn(glen, 1.0)));
            if (q == 0) {
                next[0] = o;
                for (int j = 1; j < pad4(S_); ++j) next[j] = 0.0f;
                if (live) a.states[((step + 1) * E + e) * S_] = o;
            }
        } else {
            if (!done) {  // synth17x6: component q on lane q (and 16 on lane 0)
                const double* tb = a.env.synth_b + chosen * kSynthObs;
                const double nb_a = gshfl(sq_own, (q + 1) & 15);
                const double nb_b = gshfl(s16, 0);
                const double nb = q == 15 ? nb_b : nb_a;
                const double s0 = gshfl(sq_own, 0);  // neighbour of component 16
                const double n_own = __dadd_rn(
                    sq_own, __dmul_rn(0.05, __dadd_rn(__dsub_rn(__dmul_rn(0.3, nb), __dmul_rn(0.5, sq_own)), tb[q])));
                double n16 = 0.0;
                if (q == 0)
                    n16 = __dadd_rn(s16, __dmul_rn(0.05, __dadd_rn(__dsub_rn(__dmul_rn(0.3, s0), __dmul_rn(0.5, s16)),
                                                                   tb[16])));
                const double sq2 = __dmul_rn(n_own, n_own);
                double sum = 0.0;  // sequential in component order (bit-exact reward)
                for (int c = 0; c < 16; ++c) sum = __dadd_rn(sum, gshfl(sq2, c));
                sum = __dadd_rn(sum, gshfl(__dmul_rn(n16, n16), 0));
                double m = n_own < 0.0 ? -n_own : n_own;
                if (q == 0) m = dmaxd(m, n16 < 0.0 ? -n16 : n16);
#pragma unroll
                for (int off = 8; off > 0; off >>= 1) m = dmaxd(m, __shfl_xor_sync(kFull, m, off, kPerEnv));
                sq_own = n_own;
                s16 = n16;
                rew = __dsub_rn(1.0, __ddiv_rn(sum, static_cast<double>(kSynthObs)));
                d = m > 2.0;
            }
            const float o = static_cast<float>(sq_own);
            next[q] = o;
            if (q == 0) {
                next[16] = static_cast<float>(s16);
                for (int j = 17; j < pad4(S_); ++j) next[j] = 0.0f;
            }
            if (live) {
                float* nt = a.states + ((step + 1) * E + e) * S_;
                nt[q] = o;
                if (q == 0) nt[16] = static_cast<float>(s16);
            }
        }
        if (!done) {
            if (a.env.max_steps > 0 && stepc + 1 >= a.env.max_steps) d = true;
            stepc += 1;
        }
        if (live && q == 0) {
            a.reward[ti] = done ? 0.0f : static_cast<float>(rew);
            a.done_f[ti] = (done || d) ? 1.0f : 0.0f;
            a.reward_d[ti] = done ? 0.0 : rew;
        }
        done = done || d;
        __syncthreads();
        // the next step's input must sit in buffer 0: copy if the layer count left it in 1
        if ((cur ^ 1) != 0) {
            float* h0w = reinterpret_cast<float*>(smem + S.h[0]) + r * kHStride;
            for (int j = q; j < pad4(S_); j += kPerEnv) h0w[j] = next[j];
            __syncthreads();
        }
    }
    if (live) {
        if (ENV == 0) {
            if (q == 0) {
                a.est[e] = gx;
                a.est[E + e] = glen;
            }
        } else {
            a.est[q * E + e] = sq_own;
            if (q == 0) a.est[16 * E + e] = s16;
        }
        if (q == 0) {
            a.done[e] = done ? 1 : 0;
            a.stepc[e] = stepc;
        }
    }
}

}  // namespace

size_t fast_rollout_smem_bytes(const FastRolloutArgs& a) { return rollout_carve(a).total; }

void fast_rollout(cudaStream_t s, const DeviceCtx* ctx, const FastRolloutArgs& a) {
    const size_t smem = rollout_carve(a).total;
    const unsigned grid = static_cast<unsigned>((a.E + kEnvsPerCta - 1) / kEnvsPerCta);
    if (a.env.kind == 0) {
        FLW_CUDA(cudaFuncSetAttribute(k_rollout_episode<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k_rollout_episode<0><<<grid, kThreads, smem, s>>>(ctx, a);
    } else {
        FLW_CUDA(cudaFuncSetAttribute(k_rollout_episode<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k_rollout_episode<1><<<grid, kThreads, smem, s>>>(ctx, a);
    }
}

}  // namespace flw
