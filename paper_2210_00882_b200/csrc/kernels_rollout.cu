// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 32 envs for
// the whole episode; per step it runs
//   policy MLP   on the tensor cores with f32 accuracy: mma.sync m16n8k8 TF32 in the 3xTF32 split
//                (x = hi + lo; x.w ~ lo.hi + hi.lo + hi.hi, f32 accumulate), so the logits keep
//                ~2^-20 relative error. Warp w owns env rows [16(w%2), +16) and output tiles w/2
//                and w/2 + 4 of every layer (8 warps for 32 envs); activations and W^T in shared
//                memory with row strides = 4 (mod 32) (conflict-free fragment loads)
//   PolicyApply  one thread per env (warp 0): the reference's double-precision softmax /
//                inverse-CDF sampling on the f32 logits (interp.cpp:175-203)
//   EnvStep      same thread, env state in its registers, bit-exact double dynamics (envs.cuh)
//   trajectory   written in place, t-major (the learn phase reads it without copies)
// with the policy weights staged in shared memory once and no HBM round trip of env state or
// activations between steps. The rollout is a chain of T x L dependent layers over only 32 envs
// per CTA, so it is latency-bound: a tcgen05 tile (M >= 64 rows per CTA, TMEM round trip per
// layer) would idle more than half the SMs at E = 4096; the warp-level MMA keeps all CTAs busy.
#include <cuda_runtime.h>

#include "common.cuh"
#include "engine.hpp"
#include "fast.cuh"

namespace flw {

namespace {

#ifndef FLW_ROLLOUT_EPC
#define FLW_ROLLOUT_EPC 32
#endif
constexpr int kEnvsPerCta = FLW_ROLLOUT_EPC;  // 16 or 32 (A/B: -DFLW_ROLLOUT_EPC=16)
constexpr int kMT = kEnvsPerCta / 16;          // 16-row MMA tiles of envs
constexpr int kWarps = 4 * kMT;                // warp (mt, nt0): output tiles nt0 and nt0 + 4
constexpr int kThreads = 32 * kWarps;
constexpr int kHStride = 68;  // hidden activation row stride (floats): >= 64, = 4 (mod 32)

__host__ __device__ inline int pad8(int x) { return (x + 7) & ~7; }
// row stride (floats) of a [rows x k] f32 matrix read as MMA fragments: >= pad8(k), = 4 (mod 32)
__host__ __device__ inline int kstride(int k) { return ((pad8(k) + 31) & ~31) + 4; }

struct RolloutSmem {
    uint32_t w[kMaxLayers], b[kMaxLayers], x, h[2], total;
};

// W_l^T stored [pad8(out) x kstride(in)] (zero padded): row n = the weights of output n.
__host__ __device__ inline RolloutSmem rollout_carve(const FastRolloutArgs& a) {
    RolloutSmem s{};
    uint32_t off = 0;
    for (int l = 0; l < a.L; ++l) {
        s.w[l] = off;
        off += static_cast<uint32_t>(pad8(a.dims[l + 1]) * kstride(a.dims[l]) * 4);
        s.b[l] = off;
        off += static_cast<uint32_t>(pad8(a.dims[l + 1]) * 4);
    }
    s.x = off;
    off += static_cast<uint32_t>(kEnvsPerCta * kstride(a.dims[0]) * 4);
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

// x = hi + lo: hi = x truncated to TF32 (19 bits), lo = x - hi exactly (|lo| < 2^-10 |x|); the
// tensor core reads lo's top 19 bits, so x is carried to ~2^-20 relative. Two instructions
// (cvt.rna.tf32.f32 is a 4-instruction sequence on sm_100a).
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = __float_as_uint(x) & 0xFFFFE000u;
    lo = __float_as_uint(x - __uint_as_float(hi));
}

__device__ __forceinline__ void mma_tf32(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// acc += A[16 x 8] . W^T tile (8 outputs) in 3xTF32; A fragment already split.
__device__ __forceinline__ void mma3(float* acc, const uint32_t* ahi, const uint32_t* alo, const float* wrow,
                                     int kc) {
    uint32_t bhi[2], blo[2];
    split_tf32(wrow[kc], bhi[0], blo[0]);
    split_tf32(wrow[kc + 4], bhi[1], blo[1]);
    mma_tf32(acc, alo, bhi);
    mma_tf32(acc, ahi, blo);
    mma_tf32(acc, ahi, bhi);
}

template <int ENV>
__global__ void __launch_bounds__(kThreads) k_rollout_episode(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const RolloutSmem S = rollout_carve(a);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t E = a.E, e0 = static_cast<int64_t>(blockIdx.x) * kEnvsPerCta;
    const int S_ = a.S, A = a.A;
    const int xs = kstride(a.dims[0]);
    // weights: W_l^T [pad8(out) x kstride(in)], zero padded
    for (int l = 0; l < a.L; ++l) {
        const int in = a.dims[l], out = a.dims[l + 1], ks = kstride(in), op = pad8(out);
        float* W = reinterpret_cast<float*>(smem + S.w[l]);
        float* B = reinterpret_cast<float*>(smem + S.b[l]);
        for (int i = t; i < op * ks; i += kThreads) {
            const int o = i / ks, ii = i % ks;
            W[i] = (o < out && ii < in) ? a.params[a.woff[l] + ii * out + o] : 0.0f;
        }
        for (int o = t; o < op; o += kThreads) B[o] = o < out ? a.params[a.boff[l] + o] : 0.0f;
    }
    // zero the activation buffers once: padded input columns must read as 0
    for (int i = t; i < kEnvsPerCta * xs + 2 * kEnvsPerCta * kHStride; i += kThreads)
        reinterpret_cast<float*>(smem + S.x)[i] = 0.0f;
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
    float* xb = reinterpret_cast<float*>(smem + S.x);
    if (live) {
#pragma unroll
        for (int j = 0; j < SW; ++j) st[j] = a.est[j * E + e];
        done = a.done[e] != 0;
        stepc = a.stepc[e];
        for (int j = 0; j < S_; ++j) xb[t * xs + j] = a.states[(a.step0 * E + e) * S_ + j];
    }
    __syncthreads();
    const uint64_t ep = static_cast<uint64_t>(ctx->episode);
    const int mt = warp % kMT, nt0 = warp / kMT;
    const int ar = 16 * mt + (lane >> 2), ac = lane & 3;  // fragment row / k-column of this lane

#ifdef FLW_LEARN_TRACE
    long long tr0[8], tr1[8], tr2[8];
#endif
    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr0[step - a.step0] = clock64();
#endif
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], KT = pad8(in) / 8, NT = pad8(out) / 8;
            const float* Ain = l == 0 ? xb : reinterpret_cast<const float*>(smem + S.h[(l - 1) & 1]);
            const int as = l == 0 ? xs : kHStride;
            const float* W = reinterpret_cast<const float*>(smem + S.w[l]);
            const float* B = reinterpret_cast<const float*>(smem + S.b[l]);
            float* Out = reinterpret_cast<float*>(smem + S.h[l & 1]);
            const int ws = kstride(in);
            const bool last = l + 1 == a.L;
            if (nt0 < NT) {
                const bool two = nt0 + 4 < NT;
                float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
                const float* w0 = W + (8 * nt0 + (lane >> 2)) * ws + ac;
                const float* w1 = w0 + 32 * ws;
                const float* a0 = Ain + ar * as + ac;
#pragma unroll 4
                for (int k = 0; k < KT; ++k) {
                    uint32_t ahi[4], alo[4];
                    split_tf32(a0[8 * k], ahi[0], alo[0]);
                    split_tf32(a0[8 * k + 8 * as], ahi[1], alo[1]);
                    split_tf32(a0[8 * k + 4], ahi[2], alo[2]);
                    split_tf32(a0[8 * k + 8 * as + 4], ahi[3], alo[3]);
                    mma3(acc0, ahi, alo, w0, 8 * k);
                    if (two) mma3(acc1, ahi, alo, w1, 8 * k);
                }
                auto store = [&](const float* acc, int nt) {
                    const int n = 8 * nt + 2 * ac;
                    const float b0 = B[n], b1 = B[n + 1];
                    float v[4] = {acc[0] + b0, acc[1] + b1, acc[2] + b0, acc[3] + b1};
                    if (!last) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) v[j] = a.act == 0 ? tanh_mufu(v[j]) : fmaxf(v[j], 0.0f);
                    }
                    *reinterpret_cast<float2*>(Out + ar * kHStride + n) = make_float2(v[0], v[1]);
                    *reinterpret_cast<float2*>(Out + (ar + 8) * kHStride + n) = make_float2(v[2], v[3]);
                };
                store(acc0, nt0);
                if (two) store(acc1, nt0 + 4);
            }
            __syncthreads();
        }
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr1[step - a.step0] = clock64();
#endif
        // ---- PolicyApply + EnvStep: one owner thread per env
        if (owner) {
            const float* logits = reinterpret_cast<const float*>(smem + S.h[(a.L - 1) & 1]) + t * kHStride;
            float* h0w = xb + t * xs;  // next layer-0 input
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
