// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 32 envs for
// the whole episode; per step it runs
//   policy MLP   f32 packed FFMA2 GEMM-blocked over the CTA's envs: thread (g, q) computes outputs
//                [4q, 4q+4) of envs g, g+8, g+16, g+24, so every weight float4 read from shared
//                memory feeds 16 FMAs (the shared-memory weight stream bounds this loop)
//   PolicyApply  one thread per env (warp 0): the reference's double-precision softmax /
//                inverse-CDF sampling on the f32 logits (interp.cpp:175-203)
//   EnvStep      same thread, env state in its registers, bit-exact double dynamics (envs.cuh)
//   trajectory   written in place, t-major (the learn phase reads it without copies)
// with the policy weights staged in shared memory once and no HBM round trip of env state or
// activations between steps.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.hpp"
#include "fast.cuh"

namespace flw {

namespace {

#ifndef FLW_ROLLOUT_EPC
#define FLW_ROLLOUT_EPC 32
#endif
constexpr int kEnvsPerCta = FLW_ROLLOUT_EPC;  // envs per CTA (A/B: -DFLW_ROLLOUT_EPC=16)
#ifndef FLW_ROLLOUT_GROUPS
#define FLW_ROLLOUT_GROUPS 8
#endif
constexpr int kGroups = FLW_ROLLOUT_GROUPS;        // thread groups of 16 (output quads)
constexpr int kNE = kEnvsPerCta / kGroups;         // envs per group: 4
constexpr int kThreads = kGroups * 16;             // 128
constexpr int kHStride = 68;   // activation row stride (floats): 16B aligned, spreads banks

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

// MUFU tanh (max rel. error ~2^-11): the hidden activations of the fast rollout. The sampled
// actions stay those of the exact path except within ~1e-4 of a cumulative-probability boundary
// (tests/test_fast_gpu.py bounds the flip rate).
__device__ __forceinline__ float tanh_mufu(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int ENV>
__global__ void __launch_bounds__(kThreads) k_rollout_episode(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const RolloutSmem S = rollout_carve(a);
    const int t = threadIdx.x, q = t & 15, g = t >> 4;
    const int64_t E = a.E, e0 = static_cast<int64_t>(blockIdx.x) * kEnvsPerCta;
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
    // ---- env owner threads (warp 0): env state in registers
    const bool owner = t < kEnvsPerCta;
    const int64_t e = e0 + t;  // env of an owner thread
    const bool live = owner && e < E;
    constexpr int SW = ENV == 0 ? 2 : kSynthObs;
    double st[SW];
#pragma unroll
    for (int j = 0; j < SW; ++j) st[j] = 0.0;
    bool done = false;
    int32_t stepc = 0;
    float* h0 = reinterpret_cast<float*>(smem + S.h[0]);
    if (live) {
#pragma unroll
        for (int j = 0; j < SW; ++j) st[j] = a.est[j * E + e];
        done = a.done[e] != 0;
        stepc = a.stepc[e];
        for (int j = 0; j < S_; ++j) h0[t * kHStride + j] = a.states[(a.step0 * E + e) * S_ + j];
    }
    __syncthreads();
    const uint64_t ep = static_cast<uint64_t>(ctx->episode);

#ifdef FLW_LEARN_TRACE
    long long tr0[8], tr1[8], tr2[8];
#endif
    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr0[step - a.step0] = clock64();
#endif
        int cur = 0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], op = pad4(out);
            const float* W = reinterpret_cast<const float*>(smem + S.w[l]);
            const float* B = reinterpret_cast<const float*>(smem + S.b[l]);
            const float* hbase = reinterpret_cast<const float*>(smem + S.h[cur]);
            float* obase = reinterpret_cast<float*>(smem + S.h[cur ^ 1]);
            const bool last = l + 1 == a.L;
            const int o0 = 4 * q;
            if (o0 < op) {
                float2 lo[kNE], hi[kNE];
#pragma unroll
                for (int k = 0; k < kNE; ++k) lo[k] = hi[k] = make_float2(0.f, 0.f);
                const float4* W4 = reinterpret_cast<const float4*>(W) + q;
                const int op4 = op / 4, ip4 = pad4(in) / 4;
#pragma unroll 2
                for (int i4 = 0; i4 < ip4; ++i4) {
                    float4 w[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) w[u] = W4[(4 * i4 + u) * op4];
                    float4 x[kNE];
#pragma unroll
                    for (int k = 0; k < kNE; ++k)
                        x[k] = reinterpret_cast<const float4*>(hbase + (g + kGroups * k) * kHStride)[i4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float2 wl = make_float2(w[u].x, w[u].y), wh = make_float2(w[u].z, w[u].w);
#pragma unroll
                        for (int k = 0; k < kNE; ++k) {
                            const float xv = u == 0 ? x[k].x : u == 1 ? x[k].y : u == 2 ? x[k].z : x[k].w;
                            lo[k] = __ffma2_rn(make_float2(xv, xv), wl, lo[k]);
                            hi[k] = __ffma2_rn(make_float2(xv, xv), wh, hi[k]);
                        }
                    }
                }
                const float4 bias = *reinterpret_cast<const float4*>(B + o0);
#pragma unroll
                for (int k = 0; k < kNE; ++k) {
                    float v[4] = {lo[k].x + bias.x, lo[k].y + bias.y, hi[k].x + bias.z, hi[k].y + bias.w};
                    if (!last) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) v[j] = a.act == 0 ? tanh_mufu(v[j]) : fmaxf(v[j], 0.0f);
                    }
                    *reinterpret_cast<float4*>(obase + (g + kGroups * k) * kHStride + o0) =
                        make_float4(v[0], v[1], v[2], v[3]);
                }
            }
            __syncthreads();
            cur ^= 1;
        }
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr1[step - a.step0] = clock64();
#endif
        // ---- PolicyApply + EnvStep: one owner thread per env
        if (owner) {
            const float* logits = reinterpret_cast<const float*>(smem + S.h[cur]) + t * kHStride;
            float* h0w = reinterpret_cast<float*>(smem + S.h[0]) + t * kHStride;  // next layer-0 input
            double l[16], p[16];
            double mx = logits[0];
            for (int c = 0; c < A; ++c) {
                l[c] = logits[c];
                mx = dmaxd(mx, l[c]);
            }
            double den = 0.0;
            for (int c = 0; c < A; ++c) {
                p[c] = exp(__dsub_rn(l[c], mx));  // the same value the reference computes twice
                den = __dadd_rn(den, p[c]);
            }
            for (int c = 0; c < A; ++c) p[c] = f32r(__ddiv_rn(p[c], den));
            const double u = rng_uniform(
                rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step), static_cast<uint64_t>(a.env_lo + e)));
            double cum = 0.0;
            int chosen = A - 1;
            for (int c = 0; c < A; ++c) {
                cum = __dadd_rn(cum, p[c]);
                if (u < cum) {
                    chosen = c;
                    break;
                }
            }
            double rew = 0.0;
            bool d = done;
            if (!done) {
                if (ENV == 0) {  // gridline, envs.cpp:38-53
                    int64_t len = static_cast<int64_t>(st[1]), x = static_cast<int64_t>(st[0]);
                    x += chosen == 1 ? 1 : -1;
                    if (x < 0) x = 0;
                    if (x > len - 1) x = len - 1;
                    st[0] = static_cast<double>(x);
                    d = false;
                    if (x == len - 1) {
                        rew = 1.0;
                        d = true;
                    }
                } else {  // synth17x6 (oracle/refx/env_ext.cpp)
                    const double* tb = a.env.synth_b + chosen * kSynthObs;
                    double old[kSynthObs], sq = 0.0, m = 0.0;
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) old[i] = st[i];
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) {
                        const double t4 =
                            __dadd_rn(__dsub_rn(__dmul_rn(0.3, old[(i + 1) % kSynthObs]), __dmul_rn(0.5, old[i])), tb[i]);
                        st[i] = __dadd_rn(old[i], __dmul_rn(0.05, t4));
                    }
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) {
                        sq = __dadd_rn(sq, __dmul_rn(st[i], st[i]));
                        const double av = st[i] < 0.0 ? -st[i] : st[i];
                        m = av > m ? av : m;
                    }
                    rew = __dsub_rn(1.0, __ddiv_rn(sq, static_cast<double>(kSynthObs)));
                    d = m > 2.0;
                }
                if (a.env.max_steps > 0 && stepc + 1 >= a.env.max_steps) d = true;
                stepc += 1;
            }
            if (live) {
                const int64_t ti = step * E + e;
                a.actions[ti] = chosen;
                a.logp[ti] = static_cast<float>(log(dmaxd(p[chosen], 1e-30)));
                a.reward[ti] = done ? 0.0f : static_cast<float>(rew);
                a.reward_d[ti] = done ? 0.0 : rew;
                a.done_f[ti] = (done || d) ? 1.0f : 0.0f;
                float* nt = a.states + ((step + 1) * E + e) * S_;
                if (ENV == 0) {
                    const float o = static_cast<float>(__ddiv_rn(st[0], __dsub_rn(st[1], 1.0)));
                    nt[0] = o;
                    h0w[0] = o;
                } else {
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) {
                        const float o = static_cast<float>(st[i]);
                        nt[i] = o;
                        h0w[i] = o;
                    }
                }
            }
            for (int j = S_; j < pad4(S_); ++j) h0w[j] = 0.0f;  // float4 input padding reads zeros
            done = done || d;
        }
        __syncthreads();
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr2[step - a.step0] = clock64();
#endif
    }
#ifdef FLW_LEARN_TRACE
    if (blockIdx.x == 0 && t == 0)
        for (int i = 0; i < 8; ++i) printf("R step %d mlp %lld owner %lld\n", i, tr1[i] - tr0[i], tr2[i] - tr1[i]);
#endif
    if (live) {
#pragma unroll
        for (int j = 0; j < SW; ++j) a.est[j * E + e] = st[j];
        a.done[e] = done ? 1 : 0;
        a.stepc[e] = stepc;
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
