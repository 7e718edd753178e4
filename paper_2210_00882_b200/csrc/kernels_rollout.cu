// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 32 envs for
// the whole episode; per step it runs
//   policy MLP   on the tensor cores with f32 accuracy: mma.sync m16n8k16 F16 in a 3-term split
//                (x = hi + lo, hi = f16(x), lo = f16(x - hi), carrying ~22 significant bits;
//                x.w ~ lo.hi + hi.lo + hi.hi with f32 accumulation). Weights are split once per
//                launch and activations when they are produced, so the MMA loop only loads
//                fragments. Warp w owns env rows [16(w%2), +16) and output tiles w/2, w/2 + 4 of
//                every layer (8 warps for 32 envs); fragment row strides = 8 (mod 64) halves
//                (conflict-free loads). Valid for |activations|, |obs|, |weights| < 65504 (f16).
//   PolicyApply  one thread per env (warp 0): the reference's double-precision softmax /
//                inverse-CDF sampling on the f32 logits (interp.cpp:175-203)
//   EnvStep      same thread, env state in its registers, bit-exact double dynamics (envs.cuh)
//   trajectory   written in place, t-major (the learn phase reads it without copies)
// with the policy weights staged in shared memory once and no HBM round trip of env state or
// activations between steps. The rollout is a chain of T x L dependent layers over only 32 envs
// per CTA, so it is latency-bound: a tcgen05 tile (M >= 64 rows per CTA, TMEM round trip per
// layer) would idle more than half the SMs at E = 4096; the warp-level MMA keeps all CTAs busy.
// The legacy MMA issues at <= 0.5 instructions/clk per SM for both m16n8k8 TF32 and m16n8k16
// F16 (profiles/r01_mma_sync_rate.txt), so the F16 split does the same work in half the MMAs.
#include <cuda_fp16.h>
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
constexpr int kLStride = 20;  // f32 logits row stride (floats, >= 16)

__host__ __device__ inline int pad8(int x) { return (x + 7) & ~7; }
__host__ __device__ inline int pad16(int x) { return (x + 15) & ~15; }
// row stride (halves) of an f16 [rows x k] matrix read as MMA fragments: >= pad16(k), = 8 (mod 64)
__host__ __device__ inline int hstride(int k) { return ((pad16(k) + 63) & ~63) + 8; }

struct RolloutSmem {
    uint32_t whi[kMaxLayers], wlo[kMaxLayers], b[kMaxLayers];
    uint32_t xhi, xlo, hhi[2], hlo[2], logits, total;
};

// W_l^T as f16 hi / lo [pad8(out) x hstride(in)] (zero padded): row n = the weights of output n.
__host__ __device__ inline RolloutSmem rollout_carve(const FastRolloutArgs& a) {
    RolloutSmem s{};
    uint32_t off = 0;
    for (int l = 0; l < a.L; ++l) {
        const uint32_t wb = static_cast<uint32_t>(pad8(a.dims[l + 1]) * hstride(a.dims[l]) * 2);
        s.whi[l] = off;
        off += wb;
        s.wlo[l] = off;
        off += wb;
        s.b[l] = off;
        off += static_cast<uint32_t>(pad8(a.dims[l + 1]) * 4);
    }
    const uint32_t xb = static_cast<uint32_t>(kEnvsPerCta * hstride(a.dims[0]) * 2);
    s.xhi = off;
    off += xb;
    s.xlo = off;
    off += xb;
    int hmax = 8;
    for (int l = 1; l < a.L; ++l) hmax = a.dims[l] > hmax ? a.dims[l] : hmax;
    const uint32_t hb = static_cast<uint32_t>(kEnvsPerCta * hstride(hmax) * 2);
    for (int i = 0; i < 2; ++i) {
        s.hhi[i] = off;
        off += hb;
        s.hlo[i] = off;
        off += hb;
    }
    s.logits = off;
    off += kEnvsPerCta * kLStride * 4;
    s.total = off;
    return s;
}

// MUFU tanh (max rel. error ~2^-11): the hidden activations of the fast rollout. The sampled
// actions stay those of the exact path except within ~1e-4 of a cumulative-probability boundary
// (tests/test_fast_gpu.py bounds the flip rate).
__device__ __forceinline__ float tanh_mufu(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// (x0, x1) -> f16x2 hi = rn(x), lo = rn(x - hi)
__device__ __forceinline__ void split_f16x2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
    const __half2 h = __floats2half2_rn(x0, x1);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(x0 - hf.x, x1 - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

__device__ __forceinline__ void mma_f16(float* d, const uint32_t* a, const uint32_t* b) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int ENV>
__global__ void __launch_bounds__(kThreads) k_rollout_episode(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const RolloutSmem S = rollout_carve(a);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int64_t E = a.E, e0 = static_cast<int64_t>(blockIdx.x) * kEnvsPerCta;
    const int S_ = a.S, A = a.A;
    const int xs = hstride(a.dims[0]);
    int hmax = 8;
    for (int l = 1; l < a.L; ++l) hmax = a.dims[l] > hmax ? a.dims[l] : hmax;
    const int hs = hstride(hmax);
    // weights: W_l^T [pad8(out) x hstride(in)] f16 hi / lo, zero padded (split once per launch)
    for (int l = 0; l < a.L; ++l) {
        const int in = a.dims[l], out = a.dims[l + 1], ks = hstride(in), op = pad8(out);
        __half* Wh = reinterpret_cast<__half*>(smem + S.whi[l]);
        __half* Wl = reinterpret_cast<__half*>(smem + S.wlo[l]);
        float* B = reinterpret_cast<float*>(smem + S.b[l]);
        for (int i = t; i < op * ks; i += kThreads) {
            const int o = i / ks, ii = i % ks;
            const float w = (o < out && ii < in) ? a.params[a.woff[l] + ii * out + o] : 0.0f;
            const __half h = __float2half_rn(w);
            Wh[i] = h;
            Wl[i] = __float2half_rn(w - __half2float(h));
        }
        for (int o = t; o < op; o += kThreads) B[o] = o < out ? a.params[a.boff[l] + o] : 0.0f;
    }
    // zero the activation buffers once: padded input columns must read as 0
    for (uint32_t i = t; i < (S.logits - S.xhi) / 4; i += kThreads) reinterpret_cast<uint32_t*>(smem + S.xhi)[i] = 0u;
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
    __half* xhi = reinterpret_cast<__half*>(smem + S.xhi);
    __half* xlo = reinterpret_cast<__half*>(smem + S.xlo);
    auto put_obs = [&](int j, float o) {  // next layer-0 input, split
        const __half h = __float2half_rn(o);
        xhi[t * xs + j] = h;
        xlo[t * xs + j] = __float2half_rn(o - __half2float(h));
    };
    if (live) {
#pragma unroll
        for (int j = 0; j < SW; ++j) st[j] = a.est[j * E + e];
        done = a.done[e] != 0;
        stepc = a.stepc[e];
        for (int j = 0; j < S_; ++j) put_obs(j, a.states[(a.step0 * E + e) * S_ + j]);
    }
    __syncthreads();
    const uint64_t ep = static_cast<uint64_t>(ctx->episode);
    const int mt = warp % kMT, nt0 = warp / kMT;
    const int g8 = lane >> 2, c4 = lane & 3;
    const int ar = 16 * mt + g8;  // fragment row of this lane (and ar + 8)

#ifdef FLW_LEARN_TRACE
    long long tr0[8], tr1[8], tr2[8];
#endif
    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr0[step - a.step0] = clock64();
#endif
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], KT = pad16(in) / 16, NT = pad8(out) / 8;
            const bool first = l == 0, last = l + 1 == a.L;
            const uint32_t* Ahi = reinterpret_cast<const uint32_t*>(smem + (first ? S.xhi : S.hhi[(l - 1) & 1]));
            const uint32_t* Alo = reinterpret_cast<const uint32_t*>(smem + (first ? S.xlo : S.hlo[(l - 1) & 1]));
            const int as2 = (first ? xs : hs) / 2;  // row stride in 32-bit words
            const int ws2 = hstride(in) / 2;
            const uint32_t* Whi = reinterpret_cast<const uint32_t*>(smem + S.whi[l]);
            const uint32_t* Wlo = reinterpret_cast<const uint32_t*>(smem + S.wlo[l]);
            const float* B = reinterpret_cast<const float*>(smem + S.b[l]);
            if (nt0 < NT) {
                const bool two = nt0 + 4 < NT;
                float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
                const int aoff = ar * as2 + c4, w0off = (8 * nt0 + g8) * ws2 + c4, w1off = w0off + 32 * ws2;
#pragma unroll 2
                for (int k = 0; k < KT; ++k) {
                    const int ko = 8 * k;  // 16 halves = 8 words
                    const uint32_t ahi[4] = {Ahi[aoff + ko], Ahi[aoff + ko + 8 * as2], Ahi[aoff + ko + 4],
                                             Ahi[aoff + ko + 8 * as2 + 4]};
                    const uint32_t alo[4] = {Alo[aoff + ko], Alo[aoff + ko + 8 * as2], Alo[aoff + ko + 4],
                                             Alo[aoff + ko + 8 * as2 + 4]};
                    const uint32_t bhi[2] = {Whi[w0off + ko], Whi[w0off + ko + 4]};
                    const uint32_t blo[2] = {Wlo[w0off + ko], Wlo[w0off + ko + 4]};
                    mma_f16(acc0, alo, bhi);
                    mma_f16(acc0, ahi, blo);
                    mma_f16(acc0, ahi, bhi);
                    if (two) {
                        const uint32_t chi[2] = {Whi[w1off + ko], Whi[w1off + ko + 4]};
                        const uint32_t clo[2] = {Wlo[w1off + ko], Wlo[w1off + ko + 4]};
                        mma_f16(acc1, alo, chi);
                        mma_f16(acc1, ahi, clo);
                        mma_f16(acc1, ahi, chi);
                    }
                }
                auto store = [&](const float* acc, int nt) {
                    const int n = 8 * nt + 2 * c4;
                    const float b0 = B[n], b1 = B[n + 1];
                    float v[4] = {acc[0] + b0, acc[1] + b1, acc[2] + b0, acc[3] + b1};
                    if (last) {  // f32 logits for the owner threads
                        float* lg = reinterpret_cast<float*>(smem + S.logits);
                        *reinterpret_cast<float2*>(lg + ar * kLStride + n) = make_float2(v[0], v[1]);
                        *reinterpret_cast<float2*>(lg + (ar + 8) * kLStride + n) = make_float2(v[2], v[3]);
                        return;
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) v[j] = a.act == 0 ? tanh_mufu(v[j]) : fmaxf(v[j], 0.0f);
                    uint32_t* Ohi = reinterpret_cast<uint32_t*>(smem + S.hhi[l & 1]);
                    uint32_t* Olo = reinterpret_cast<uint32_t*>(smem + S.hlo[l & 1]);
                    const int o2 = n / 2;
                    split_f16x2(v[0], v[1], Ohi[ar * (hs / 2) + o2], Olo[ar * (hs / 2) + o2]);
                    split_f16x2(v[2], v[3], Ohi[(ar + 8) * (hs / 2) + o2], Olo[(ar + 8) * (hs / 2) + o2]);
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
            // softmax in f32 (the reference's is double, rounded to f32: the probabilities differ
            // by <= ~1 f32 ulp, far below the f32-logit deviation the fast path already has);
            // the draw and the inverse-CDF walk are the reference's (double u, double cumsum)
            const float* logits = reinterpret_cast<const float*>(smem + S.logits) + t * kLStride;
            float p[16];
            float mx = logits[0];
            for (int c = 1; c < A; ++c) mx = fmaxf(mx, logits[c]);
            float den = 0.0f;
            for (int c = 0; c < A; ++c) {
                p[c] = __expf(logits[c] - mx);
                den += p[c];
            }
            const float rden = 1.0f / den;
            for (int c = 0; c < A; ++c) p[c] *= rden;
            const double u = rng_uniform(
                rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step), static_cast<uint64_t>(a.env_lo + e)));
            double cum = 0.0;
            int chosen = A - 1;
            for (int c = 0; c < A; ++c) {
                cum = __dadd_rn(cum, static_cast<double>(p[c]));
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
                a.logp[ti] = __logf(fmaxf(p[chosen], 1e-30f));
                a.reward[ti] = done ? 0.0f : static_cast<float>(rew);
                a.reward_d[ti] = done ? 0.0 : rew;
                a.done_f[ti] = (done || d) ? 1.0f : 0.0f;
                float* nt = a.states + ((step + 1) * E + e) * S_;
                if (ENV == 0) {
                    const float o = static_cast<float>(__ddiv_rn(st[0], __dsub_rn(st[1], 1.0)));
                    nt[0] = o;
                    put_obs(0, o);
                } else {
#pragma unroll
                    for (int i = 0; i < kSynthObs; ++i) {
                        const float o = static_cast<float>(st[i]);
                        nt[i] = o;
                        put_obs(i, o);
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
