// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 32 envs for
// the episode: env state lives in registers, the policy weights are staged in shared memory
// once, and every step runs policy MLP (f32 FMA, 4 threads per env) -> PolicyApply (the
// reference's double-precision inverse-CDF sampling on the f32 logits, interp.cpp:175-203) ->
// EnvStep (bit-exact double dynamics, envs.cuh) -> trajectory write, with no HBM round trip of
// the env state or activations between steps.
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

template <int ENV>
__global__ void __launch_bounds__(kThreads) k_rollout_episode(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const RolloutSmem S = rollout_carve(a);
    const int t = threadIdx.x, q = t & (kPerEnv - 1), r = t / kPerEnv;
    const int64_t e = static_cast<int64_t>(blockIdx.x) * kEnvsPerCta + r;
    const bool live = e < a.E;
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
    // env state -> registers of the quad leader
    constexpr int SW = ENV == 0 ? 2 : kSynthObs;
    double st[SW];
    bool done = false;
    int32_t stepc = 0;
    if (live && q == 0) {
#pragma unroll
        for (int j = 0; j < SW; ++j) st[j] = a.est[j * a.E + e];
        done = a.done[e] != 0;
        stepc = a.stepc[e];
    }
    // step-0 policy input: the reset observation (trajectory block 0)
    float* h0 = reinterpret_cast<float*>(smem + S.h[0]);
    if (q == 0)
        for (int j = 0; j < S_; ++j) h0[r * kHStride + j] = live ? a.states[(a.step0 * a.E + e) * S_ + j] : 0.0f;
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
            // env's 16 threads) feeds 16 FMAs issued as 8 packed FFMA2; in-order f32 accumulation
            const int o0 = 4 * q;
            if (o0 < op) {
                float2 lo = make_float2(0.f, 0.f), hi = lo;
                const float4* W4 = reinterpret_cast<const float4*>(W) + q;
                const float4* X4 = reinterpret_cast<const float4*>(hin);
                const int op4 = op / 4, ip4 = pad4(in) / 4;
#pragma unroll 2
                for (int i4 = 0; i4 < ip4; ++i4) {
                    const float4 x = X4[i4];
                    const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const float4 w = W4[(4 * i4 + u) * op4];
                        const float2 xx = make_float2(xs[u], xs[u]);
                        lo = __ffma2_rn(xx, make_float2(w.x, w.y), lo);
                        hi = __ffma2_rn(xx, make_float2(w.z, w.w), hi);
                    }
                }
                float v[4] = {lo.x + B[o0], lo.y + B[o0 + 1], hi.x + B[o0 + 2], hi.y + B[o0 + 3]};
                if (!last) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = a.act == 0 ? tanhf(v[j]) : fmaxf(v[j], 0.0f);
                }
                *reinterpret_cast<float4*>(hout + o0) = make_float4(v[0], v[1], v[2], v[3]);
            }
            __syncthreads();
            cur ^= 1;
        }
        // PolicyApply + EnvStep by the quad leader
        const float* logits = reinterpret_cast<const float*>(smem + S.h[cur]) + r * kHStride;
        float* next = reinterpret_cast<float*>(smem + S.h[cur ^ 1]) + r * kHStride;  // next step's layer-0 input
        if (live && q == 0) {
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
            const double u = rng_uniform(rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step),
                                                 static_cast<uint64_t>(a.env_lo + e)));
            double cum = 0.0;
            int chosen = A - 1;
            for (int c = 0; c < A; ++c) {
                cum = __dadd_rn(cum, p[c]);
                if (u < cum) {
                    chosen = c;
                    break;
                }
            }
            const int64_t ti = step * a.E + e;
            a.actions[ti] = chosen;
            a.logp[ti] = static_cast<float>(log(dmaxd(p[chosen], 1e-30)));
            double rew = 0.0;
            if (!done) {
                bool d = false;
                if (ENV == 0) {  // gridline, envs.cpp:38-53
                    int64_t len = static_cast<int64_t>(st[1]), x = static_cast<int64_t>(st[0]);
                    x += chosen == 1 ? 1 : -1;
                    if (x < 0) x = 0;
                    if (x > len - 1) x = len - 1;
                    st[0] = static_cast<double>(x);
                    if (x == len - 1) {
                        rew = 1.0;
                        d = true;
                    }
                } else {  // synth17x6
                    double old[kSynthObs], sq = 0.0, m = 0.0;
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) old[i] = st[i];
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) {
                        double t4 = __dadd_rn(__dsub_rn(__dmul_rn(0.3, old[(i + 1) % kSynthObs]), __dmul_rn(0.5, old[i])),
                                              a.env.synth_b[chosen * kSynthObs + i]);
                        double nv = __dadd_rn(old[i], __dmul_rn(0.05, t4));
                        st[i] = nv;
                        sq = __dadd_rn(sq, __dmul_rn(nv, nv));
                        double av = nv < 0.0 ? -nv : nv;
                        m = av > m ? av : m;
                    }
                    rew = __dsub_rn(1.0, __ddiv_rn(sq, static_cast<double>(kSynthObs)));
                    d = m > 2.0;
                }
                if (a.env.max_steps > 0 && stepc + 1 >= a.env.max_steps) d = true;
                stepc += 1;
                done = d;
                a.reward[ti] = static_cast<float>(rew);
                a.done_f[ti] = d ? 1.0f : 0.0f;
            } else {
                a.reward[ti] = 0.0f;
                a.done_f[ti] = 1.0f;
            }
            a.reward_d[ti] = rew;
            float* nxt_traj = a.states + ((step + 1) * a.E + e) * S_;
            for (int j = 0; j < S_; ++j) {
                float o = ENV == 0 ? static_cast<float>(__ddiv_rn(st[0], __dsub_rn(st[1], 1.0))) : static_cast<float>(st[j]);
                next[j] = o;
                nxt_traj[j] = o;
            }
            for (int j = S_; j < pad4(S_); ++j) next[j] = 0.0f;  // float4 input padding reads zeros
        } else if (q == 0) {
            for (int j = 0; j < pad4(S_); ++j) next[j] = 0.0f;
        }
        __syncthreads();
        // the next step's input must sit in buffer 0: copy if the layer count left it in 1
        if ((cur ^ 1) != 0) {
            float* h0w = reinterpret_cast<float*>(smem + S.h[0]) + r * kHStride;
            for (int j = q; j < pad4(S_); j += kPerEnv) h0w[j] = next[j];
            __syncthreads();
        }
    }
    if (live && q == 0) {
#pragma unroll
        for (int j = 0; j < SW; ++j) a.est[j * a.E + e] = st[j];
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
