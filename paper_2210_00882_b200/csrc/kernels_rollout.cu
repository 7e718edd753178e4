// Fast-numerics rollout: the whole episode's T steps in ONE launch. Each CTA owns 32 envs for
// the whole episode; per step it runs
//   policy MLP   on the tensor cores with f32 accuracy: mma.sync m16n8k16 F16 in a 3-term split
//                (x = hi + lo, hi = f16(x), lo = f16(x - hi); x.w ~ lo.hi + hi.lo + hi.hi with f32
//                accumulation). The pair carries ~22 significant bits for |x| >= 2^-3; below
//                that lo is an f16 subnormal (|lo| < 2^-14) with absolute precision 2^-24, e.g.
//                ~18 bits at |x| ~ 1e-2 (measured logp error at C2: 4.4e-6 relative). Weights are split once per
//                launch and activations when they are produced, and both live in shared memory
//                in FRAGMENT-MAJOR order ([tile][k-step][lane] x 16 B): every MMA operand is one
//                conflict-free 128-bit load. Warp w owns env rows [16(w%2), +16) and the output
//                tiles 2(w/2), 2(w/2)+1 of every layer, so its two accumulator fragments ARE the
//                next layer's A fragment for k-step w/2 (one 128-bit store each for hi and lo).
//                Valid for |activations|, |obs|, |weights| < 65504 (f16): an observation outside
//                that range poisons the step's reward (NaN) and the episode call fails loudly.
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
// fragment-major operand images (16 B per lane per fragment):
//   weights of layer l: [NT = pad8(out)/8][KT = pad16(in)/16][32 lanes] x {b0 hi, b1 hi, b0 lo, b1 lo}
//   activations:        [kMT][KT][32 lanes] x {a0..a3} for hi and for lo (separate images)
__host__ __device__ inline uint32_t wfrag_bytes(int in, int out) {
    return static_cast<uint32_t>((pad8(out) / 8) * (pad16(in) / 16) * 32 * 16);
}
__host__ __device__ inline uint32_t afrag_bytes(int k) { return static_cast<uint32_t>(kMT * (pad16(k) / 16) * 32 * 16); }

struct RolloutSmem {
    uint32_t w0, xhi, xlo, hhi[2], hlo[2], logits, sb, total;  // weights: layers back to back from w0
};

__host__ __device__ inline RolloutSmem rollout_carve(const FastRolloutArgs& a) {
    RolloutSmem s{};
    uint32_t off = 0;
    s.w0 = off;
    for (int l = 0; l < a.L; ++l) off += wfrag_bytes(a.dims[l], a.dims[l + 1]) + static_cast<uint32_t>(pad16(a.dims[l + 1]) * 4);
    s.xhi = off;
    off += afrag_bytes(a.dims[0]);
    s.xlo = off;
    off += afrag_bytes(a.dims[0]);
    int hmax = 16;
    for (int l = 1; l < a.L; ++l) hmax = a.dims[l] > hmax ? a.dims[l] : hmax;
    for (int i = 0; i < 2; ++i) {
        s.hhi[i] = off;
        off += afrag_bytes(hmax);
        s.hlo[i] = off;
        off += afrag_bytes(hmax);
    }
    s.logits = off;
    off += kEnvsPerCta * kLStride * 4;
    s.sb = off;  // synth17x6 action table B[a][i] (double)
    off += 16 * kSynthObs * 8;
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

// named barrier of env tile mt's four warps (ids 1.. ; 0 is __syncthreads)
__device__ __forceinline__ void tile_sync(int mt) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(1 + mt), "r"(128) : "memory");
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
    const int KT0 = pad16(a.dims[0]) / 16;
    // weights: fragment-major W_l^T images, f16 hi / lo (split once per launch), then the f32 bias
    {
        uint32_t off = S.w0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], NT = pad8(out) / 8, KT = pad16(in) / 16;
            uint32_t* Wf = reinterpret_cast<uint32_t*>(smem + off);
            for (int i = t; i < NT * KT * 32 * 2; i += kThreads) {  // (nt, kk, lane, fragment reg)
                const int r = i & 1, ln = (i >> 1) & 31, kk = (i >> 6) % KT, nt = (i >> 6) / KT;
                const int n = 8 * nt + (ln >> 2), k = 16 * kk + 8 * r + 2 * (ln & 3);
                float w[2];
                for (int h = 0; h < 2; ++h)
                    w[h] = (n < out && k + h < in) ? a.params[a.woff[l] + static_cast<int64_t>(k + h) * out + n] : 0.0f;
                uint32_t hi, lo;
                split_f16x2(w[0], w[1], hi, lo);
                Wf[4 * ((nt * KT + kk) * 32 + ln) + r] = hi;
                Wf[4 * ((nt * KT + kk) * 32 + ln) + 2 + r] = lo;
            }
            off += wfrag_bytes(in, out);
            float* B = reinterpret_cast<float*>(smem + off);
            for (int o = t; o < pad16(out); o += kThreads) B[o] = o < out ? a.params[a.boff[l] + o] : 0.0f;
            off += static_cast<uint32_t>(pad16(out) * 4);
        }
    }
    if (ENV == 1)
        for (int i = t; i < a.A * kSynthObs; i += kThreads)
            reinterpret_cast<double*>(smem + S.sb)[i] = a.env.synth_b[i];
    // zero the activation images once: padded input columns must read as 0
    for (uint32_t i = t; i < (S.logits - S.xhi) / 4; i += kThreads) reinterpret_cast<uint32_t*>(smem + S.xhi)[i] = 0u;
    __syncthreads();
    // ---- env owner threads: lanes 0-15 of warp mt own the 16 envs of env tile mt (state in
    // registers). The env tiles are independent pipelines (MLP -> owner -> MLP ...) that sync on
    // their own named barriers, so one tile's owner phase overlaps another tile's MLP.
    const int le = 16 * warp + lane;  // local env of an owner thread
    const bool owner = warp < kMT && lane < 16;
    const int64_t e = e0 + le;  // env of an owner thread
    const bool live = owner && e < E;
    constexpr int SW = ENV == 0 ? 2 : kSynthObs;
    double st[SW];
#pragma unroll
    for (int j = 0; j < SW; ++j) st[j] = 0.0;
    bool done = false;
    int32_t stepc = 0;
    __half* xhi = reinterpret_cast<__half*>(smem + S.xhi);
    __half* xlo = reinterpret_cast<__half*>(smem + S.xlo);
    bool f16_oob = false;  // an observation left the f16 range of the split MLP
    auto put_obs = [&](int j, float o) {  // next layer-0 input element (row t, column j), split
        const int rr = le & 15, kc = j & 15;
        const int ln = 4 * (rr & 7) + ((kc & 7) >> 1), reg = 2 * (kc >> 3) + (rr >> 3);
        const int el = 2 * (4 * (((le >> 4) * KT0 + (j >> 4)) * 32 + ln) + reg) + (kc & 1);
        f16_oob = f16_oob || !(fabsf(o) < 65504.0f);
        const __half h = __float2half_rn(o);
        xhi[el] = h;
        xlo[el] = __float2half_rn(o - __half2float(h));
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
    const int mt = warp % kMT, jw = warp / kMT;  // env tile, output tile pair (2jw, 2jw + 1)
    const int g8 = lane >> 2, c4 = lane & 3;
    const int ar = 16 * mt + g8;  // fragment row of this lane (and ar + 8)

#ifdef FLW_LEARN_TRACE
    long long tr0[8], tr1[8], tr2[8];
    long long trl[3][8];  // step 2, per layer: MMA loop done, epilogue stored, tile barrier passed
#endif
    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr0[step - a.step0] = clock64();
#endif
        // the owner's action draw (integer hashing) issues ahead of the MLP and overlaps it
        double u = 0.0;
        if (owner)
            u = rng_uniform(
                rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step), static_cast<uint64_t>(a.env_lo + e)));
        uint32_t woff = S.w0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], KT = pad16(in) / 16, NT = pad8(out) / 8;
            const bool last = l + 1 == a.L;
            const uint4* Ahi = reinterpret_cast<const uint4*>(smem + (l == 0 ? S.xhi : ((l - 1) & 1) ? S.hhi[1] : S.hhi[0]));
            const uint4* Alo = reinterpret_cast<const uint4*>(smem + (l == 0 ? S.xlo : ((l - 1) & 1) ? S.hlo[1] : S.hlo[0]));
            const uint4* Wf = reinterpret_cast<const uint4*>(smem + woff);
            const float* B = reinterpret_cast<const float*>(smem + woff + wfrag_bytes(in, out));
            woff += wfrag_bytes(in, out) + static_cast<uint32_t>(pad16(out) * 4);
            const int n0 = 2 * jw;
            if (n0 < NT) {
                const bool two = n0 + 1 < NT;
#ifdef FLW_LEARN_TRACE
                const bool trl_on = step == a.step0 + 2 && l < 8;
#endif
                float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
                const uint4* ap = Ahi + mt * KT * 32 + lane;
                const uint4* alp = Alo + mt * KT * 32 + lane;
                const uint4* w0p = Wf + n0 * KT * 32 + lane;
                const uint4* w1p = w0p + KT * 32;
#pragma unroll 4
                for (int kk = 0; kk < KT; ++kk) {
                    const uint4 ah = ap[32 * kk], al = alp[32 * kk], b0 = w0p[32 * kk];
                    const uint32_t ahv[4] = {ah.x, ah.y, ah.z, ah.w}, alv[4] = {al.x, al.y, al.z, al.w};
                    const uint32_t bh0[2] = {b0.x, b0.y}, bl0[2] = {b0.z, b0.w};
                    mma_f16(acc0, alv, bh0);
                    mma_f16(acc0, ahv, bl0);
                    mma_f16(acc0, ahv, bh0);
                    if (two) {
                        const uint4 b1 = w1p[32 * kk];
                        const uint32_t bh1[2] = {b1.x, b1.y}, bl1[2] = {b1.z, b1.w};
                        mma_f16(acc1, alv, bh1);
                        mma_f16(acc1, ahv, bl1);
                        mma_f16(acc1, ahv, bh1);
                    }
                }
#ifdef FLW_LEARN_TRACE
                if (trl_on) trl[0][l] = clock64();
#endif
                // bias, activation; output columns n0*8 + 2c (+1) and (n0 + 1)*8 + 2c (+1)
                const int na = 8 * n0 + 2 * c4, nb = na + 8;
                float v[8] = {acc0[0] + B[na], acc0[1] + B[na + 1], acc0[2] + B[na], acc0[3] + B[na + 1],
                              acc1[0] + B[nb], acc1[1] + B[nb + 1], acc1[2] + B[nb], acc1[3] + B[nb + 1]};
                if (last) {  // f32 logits for the owner threads
                    float* lg = reinterpret_cast<float*>(smem + S.logits);
                    *reinterpret_cast<float2*>(lg + ar * kLStride + na) = make_float2(v[0], v[1]);
                    *reinterpret_cast<float2*>(lg + (ar + 8) * kLStride + na) = make_float2(v[2], v[3]);
                    if (two) {
                        *reinterpret_cast<float2*>(lg + ar * kLStride + nb) = make_float2(v[4], v[5]);
                        *reinterpret_cast<float2*>(lg + (ar + 8) * kLStride + nb) = make_float2(v[6], v[7]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = a.act == 0 ? tanh_mufu(v[j]) : fmaxf(v[j], 0.0f);
                    if (!two) v[4] = v[5] = v[6] = v[7] = 0.0f;
                    // the two accumulator fragments = the next layer's A fragment of k-step jw
                    uint4 hi, lo;
                    split_f16x2(v[0], v[1], hi.x, lo.x);
                    split_f16x2(v[2], v[3], hi.y, lo.y);
                    split_f16x2(v[4], v[5], hi.z, lo.z);
                    split_f16x2(v[6], v[7], hi.w, lo.w);
                    const int KTn = pad16(out) / 16;
                    reinterpret_cast<uint4*>(smem + ((l & 1) ? S.hhi[1] : S.hhi[0]))[(mt * KTn + jw) * 32 + lane] = hi;
                    reinterpret_cast<uint4*>(smem + ((l & 1) ? S.hlo[1] : S.hlo[0]))[(mt * KTn + jw) * 32 + lane] = lo;
                }
#ifdef FLW_LEARN_TRACE
                if (trl_on) trl[1][l] = clock64();
#endif
            }
            tile_sync(mt);
#ifdef FLW_LEARN_TRACE
            if (step == a.step0 + 2 && l < 8) trl[2][l] = clock64();
#endif
        }
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr1[step - a.step0] = clock64();
#endif
        // ---- PolicyApply + EnvStep: one owner thread per env
        if (owner) {
            // softmax in f32 (the reference's is double, rounded to f32: the probabilities differ
            // by <= ~1 f32 ulp, far below the f32-logit deviation the fast path already has);
            // the draw and the inverse-CDF walk are the reference's (double u, double cumsum)
            const float* logits = reinterpret_cast<const float*>(smem + S.logits) + le * kLStride;
            // static loop bounds (predicated on A <= 16): p[] stays in registers
            float p[16];
            float mx = logits[0];
#pragma unroll
            for (int c = 1; c < 16; ++c)
                if (c < A) mx = fmaxf(mx, logits[c]);
            float den = 0.0f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                p[c] = c < A ? __expf(logits[c] - mx) : 0.0f;
                den += p[c];
            }
            const float rden = 1.0f / den;
#pragma unroll
            for (int c = 0; c < 16; ++c) p[c] *= rden;
            double cum = 0.0;
            int chosen = A - 1;
            float pch = 0.0f;  // p[chosen]
            bool found = false;
#pragma unroll
            for (int c = 0; c < 16; ++c) {  // the first c with u < cumsum (interp.cpp:175-203)
                if (c < A && !found) {
                    cum = __dadd_rn(cum, static_cast<double>(p[c]));
                    if (u < cum) {
                        chosen = c;
                        found = true;
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c == chosen) pch = p[c];
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
                    const double* tb = reinterpret_cast<const double*>(smem + S.sb) + chosen * kSynthObs;
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
                a.logp[ti] = __logf(fmaxf(pch, 1e-30f));
                a.reward[ti] = done ? 0.0f : static_cast<float>(rew);
                a.reward_d[ti] = f16_oob ? __longlong_as_double(0x7ff8000000000000LL) : (done ? 0.0 : rew);
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
        tile_sync(mt);
#ifdef FLW_LEARN_TRACE
        if (step - a.step0 < 8) tr2[step - a.step0] = clock64();
#endif
    }
#ifdef FLW_LEARN_TRACE
    if (blockIdx.x == 0 && t == 0)
        for (int i = 0; i < 8; ++i) printf("R step %d mlp %lld owner %lld\n", i, tr1[i] - tr0[i], tr2[i] - tr1[i]);
    if (blockIdx.x == 0 && t == 0)
        for (int l = 0; l < a.L && l < 8; ++l)
            printf("RL layer %d mma %lld epi %lld sync %lld\n", l, trl[0][l] - (l ? trl[2][l - 1] : tr0[2]),
                   trl[1][l] - trl[0][l], trl[2][l] - trl[1][l]);
#endif
    if (live) {
#pragma unroll
        for (int j = 0; j < SW; ++j) a.est[j * E + e] = st[j];
        a.done[e] = done ? 1 : 0;
        a.stepc[e] = stepc;
    }
}


// ------------------------------------------------------------------------------------------
// MAPPO on spread_lite, fast numerics: the whole episode in one launch, the same fragment-major
// 3-term F16 MLP over the CTA's agent-major rows r = a * EPC + le (EPC envs per CTA, n agents;
// 16-row MMA tiles, the last one zero padded), then per step
//   PolicyApply  one thread per row: f32 softmax, the reference's draw
//                U(key(seed, 0x616374, ep, step, a*env_total + env_lo + e)) and inverse-CDF walk
//   EnvStep      one thread per env: the exact spread_lite moves / rewards / done in double
//                (envs.cpp:111-150, same arithmetic as k_rollout_mappo), state in shared memory
//   emit         one thread per row: the agent observation (envs.cpp:96-109) -> next MLP input and
//                the trajectory layouts the learn phase reads (joint, prows, cin)
struct MappoSmem {
    uint32_t w0, xhi, xlo, hhi[2], hlo[2], logits, st, act, rew, dn, total;
};

__host__ __device__ inline MappoSmem mappo_carve(const FastRolloutArgs& a, int EPC) {
    MappoSmem s{};
    const int n = a.env.n_agents, MT = (n * EPC + 15) / 16;
    uint32_t off = 0;
    s.w0 = off;
    for (int l = 0; l < a.L; ++l) off += wfrag_bytes(a.dims[l], a.dims[l + 1]) + static_cast<uint32_t>(pad16(a.dims[l + 1]) * 4);
    const uint32_t xb = static_cast<uint32_t>(MT * (pad16(a.dims[0]) / 16) * 512);
    s.xhi = off;
    off += xb;
    s.xlo = off;
    off += xb;
    int hmax = 16;
    for (int l = 1; l < a.L; ++l) hmax = a.dims[l] > hmax ? a.dims[l] : hmax;
    const uint32_t hb = static_cast<uint32_t>(MT * (pad16(hmax) / 16) * 512);
    for (int i = 0; i < 2; ++i) {
        s.hhi[i] = off;
        off += hb;
        s.hlo[i] = off;
        off += hb;
    }
    s.logits = off;
    off += static_cast<uint32_t>(MT * 16 * kLStride * 4);
    s.st = off;  // env state, [4n][EPC] doubles
    off += static_cast<uint32_t>(4 * n * EPC * 8);
    s.act = off;
    off += static_cast<uint32_t>(MT * 16 * 4);
    s.rew = off;  // per-row reward of the step (double)
    off += static_cast<uint32_t>(MT * 16 * 8);
    s.dn = off;  // per-env done flag
    off += static_cast<uint32_t>(EPC * 4);
    s.total = off;
    return s;
}

template <int EPC>
__global__ void __launch_bounds__(256, 1) k_rollout_mappo_fast(const DeviceCtx* __restrict__ ctx, FastRolloutArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    const MappoSmem S = mappo_carve(a, EPC);
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int n = a.env.n_agents, A = a.A, Sd = 2 + 2 * n, W = n * Sd, C = W + n;
    const int rows = n * EPC, MT = (rows + 15) / 16;
    const int64_t E = a.E, e0 = static_cast<int64_t>(blockIdx.x) * EPC, R = static_cast<int64_t>(n) * E;
    const int KT0 = pad16(a.dims[0]) / 16;
    {  // weights, as k_rollout_episode
        uint32_t off = S.w0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], NT = pad8(out) / 8, KT = pad16(in) / 16;
            uint32_t* Wf = reinterpret_cast<uint32_t*>(smem + off);
            for (int i = t; i < NT * KT * 32 * 2; i += blockDim.x) {
                const int r = i & 1, ln = (i >> 1) & 31, kk = (i >> 6) % KT, nt = (i >> 6) / KT;
                const int nn = 8 * nt + (ln >> 2), k = 16 * kk + 8 * r + 2 * (ln & 3);
                float w[2];
                for (int h = 0; h < 2; ++h)
                    w[h] = (nn < out && k + h < in) ? a.params[a.woff[l] + static_cast<int64_t>(k + h) * out + nn] : 0.0f;
                uint32_t hi, lo;
                split_f16x2(w[0], w[1], hi, lo);
                Wf[4 * ((nt * KT + kk) * 32 + ln) + r] = hi;
                Wf[4 * ((nt * KT + kk) * 32 + ln) + 2 + r] = lo;
            }
            off += wfrag_bytes(in, out);
            float* B = reinterpret_cast<float*>(smem + off);
            for (int o = t; o < pad16(out); o += blockDim.x) B[o] = o < out ? a.params[a.boff[l] + o] : 0.0f;
            off += static_cast<uint32_t>(pad16(out) * 4);
        }
    }
    for (uint32_t i = t; i < (S.logits - S.xhi) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem + S.xhi)[i] = 0u;
    double* sts = reinterpret_cast<double*>(smem + S.st);
    int* acts = reinterpret_cast<int*>(smem + S.act);
    double* rews = reinterpret_cast<double*>(smem + S.rew);
    int* dns = reinterpret_cast<int*>(smem + S.dn);
    // env threads: t < EPC; row threads: t < rows (agent ra, local env rle)
    const bool envt = t < EPC && e0 + t < E;
    const int ra = t / EPC, rle = t % EPC;
    const int64_t re = e0 + rle;
    const bool rowt = t < rows && re < E;
    bool done = false;
    int32_t stepc = 0;
    if (envt) {
        for (int i = 0; i < 4 * n; ++i) sts[i * EPC + t] = a.est[i * E + e0 + t];
        done = a.done[e0 + t] != 0;
        stepc = a.stepc[e0 + t];
        dns[t] = done ? 1 : 0;
    }
    __syncthreads();
    __half* xhi = reinterpret_cast<__half*>(smem + S.xhi);
    __half* xlo = reinterpret_cast<__half*>(smem + S.xlo);
    // observation of row (ra, rle) from the state (envs.cpp:96-109): next MLP input, and the step
    // block `blk` of the trajectory layouts when blk >= 0
    auto emit = [&](int64_t blk) {
        const double xa = sts[(2 * ra) * EPC + rle], ya = sts[(2 * ra + 1) * EPC + rle];
        float* pr = blk >= 0 ? a.states + (blk * R + static_cast<int64_t>(ra) * E + re) * Sd : nullptr;
        float* jr = blk >= 0 ? a.joint + (blk * E + re) * W + ra * Sd : nullptr;
        for (int j = 0; j < Sd; ++j) {
            float o;
            if (j < 2) {
                o = static_cast<float>(j == 0 ? xa : ya);
            } else {
                const int lm = (j - 2) >> 1;
                o = static_cast<float>((j & 1) == 0 ? __dsub_rn(sts[(2 * n + 2 * lm) * EPC + rle], xa)
                                                   : __dsub_rn(sts[(2 * n + 2 * lm + 1) * EPC + rle], ya));
            }
            const int rr = t & 15, kc = j & 15;
            const int ln = 4 * (rr & 7) + ((kc & 7) >> 1), reg = 2 * (kc >> 3) + (rr >> 3);
            const int el = 2 * (4 * (((t >> 4) * KT0 + (j >> 4)) * 32 + ln) + reg) + (kc & 1);
            const __half h = __float2half_rn(o);
            xhi[el] = h;
            xlo[el] = __float2half_rn(o - __half2float(h));
            if (pr) {
                pr[j] = o;
                jr[j] = o;
            }
        }
        if (blk >= 0 && a.cin) {  // [joint(t, e) | one-hot(a)] (programs.cpp:390-402)
            float* cr = a.cin + (blk * R + static_cast<int64_t>(ra) * E + re) * C;
            for (int b = 0; b < n; ++b) {
                const double xb = sts[(2 * b) * EPC + rle], yb = sts[(2 * b + 1) * EPC + rle];
                cr[b * Sd] = static_cast<float>(xb);
                cr[b * Sd + 1] = static_cast<float>(yb);
                for (int lm = 0; lm < n; ++lm) {
                    cr[b * Sd + 2 + 2 * lm] = static_cast<float>(__dsub_rn(sts[(2 * n + 2 * lm) * EPC + rle], xb));
                    cr[b * Sd + 3 + 2 * lm] = static_cast<float>(__dsub_rn(sts[(2 * n + 2 * lm + 1) * EPC + rle], yb));
                }
            }
            for (int j = 0; j < n; ++j) cr[W + j] = j == ra ? 1.0f : 0.0f;
        }
    };
    if (rowt) emit(-1);  // step0's rows are in the trajectory already (reset or previous call)
    __syncthreads();
    const uint64_t ep = static_cast<uint64_t>(ctx->episode);
    const int g8 = lane >> 2, c4 = lane & 3;
    for (int64_t step = a.step0; step < a.step0 + a.nsteps; ++step) {
        double u = 0.0;
        if (rowt)
            u = rng_uniform(rng_key(a.seed, kActionStream, ep, static_cast<uint64_t>(step),
                                    static_cast<uint64_t>(ra * a.env_total + a.env_lo + re)));
        uint32_t woff = S.w0;
        for (int l = 0; l < a.L; ++l) {
            const int in = a.dims[l], out = a.dims[l + 1], KT = pad16(in) / 16, NT = pad8(out) / 8;
            const bool last = l + 1 == a.L;
            const uint4* Ahi = reinterpret_cast<const uint4*>(smem + (l == 0 ? S.xhi : ((l - 1) & 1) ? S.hhi[1] : S.hhi[0]));
            const uint4* Alo = reinterpret_cast<const uint4*>(smem + (l == 0 ? S.xlo : ((l - 1) & 1) ? S.hlo[1] : S.hlo[0]));
            const uint4* Wf = reinterpret_cast<const uint4*>(smem + woff);
            const float* B = reinterpret_cast<const float*>(smem + woff + wfrag_bytes(in, out));
            woff += wfrag_bytes(in, out) + static_cast<uint32_t>(pad16(out) * 4);
            const int KTn = pad16(out) / 16;
            for (int pi = warp; pi < MT * 4; pi += 8) {
                const int mt = pi % MT, jw = pi / MT, n0 = 2 * jw;
                if (n0 >= NT) continue;
                const bool two = n0 + 1 < NT;
                float acc0[4] = {0.f, 0.f, 0.f, 0.f}, acc1[4] = {0.f, 0.f, 0.f, 0.f};
                const uint4* ap = Ahi + mt * KT * 32 + lane;
                const uint4* alp = Alo + mt * KT * 32 + lane;
                const uint4* w0p = Wf + n0 * KT * 32 + lane;
                const uint4* w1p = w0p + KT * 32;
                for (int kk = 0; kk < KT; ++kk) {
                    const uint4 ah = ap[32 * kk], al = alp[32 * kk], b0 = w0p[32 * kk];
                    const uint32_t ahv[4] = {ah.x, ah.y, ah.z, ah.w}, alv[4] = {al.x, al.y, al.z, al.w};
                    const uint32_t bh0[2] = {b0.x, b0.y}, bl0[2] = {b0.z, b0.w};
                    mma_f16(acc0, alv, bh0);
                    mma_f16(acc0, ahv, bl0);
                    mma_f16(acc0, ahv, bh0);
                    if (two) {
                        const uint4 b1 = w1p[32 * kk];
                        const uint32_t bh1[2] = {b1.x, b1.y}, bl1[2] = {b1.z, b1.w};
                        mma_f16(acc1, alv, bh1);
                        mma_f16(acc1, ahv, bl1);
                        mma_f16(acc1, ahv, bh1);
                    }
                }
                const int na = 8 * n0 + 2 * c4, nb = na + 8, ar = 16 * mt + g8;
                float v[8] = {acc0[0] + B[na], acc0[1] + B[na + 1], acc0[2] + B[na], acc0[3] + B[na + 1],
                              acc1[0] + B[nb], acc1[1] + B[nb + 1], acc1[2] + B[nb], acc1[3] + B[nb + 1]};
                if (last) {
                    float* lg = reinterpret_cast<float*>(smem + S.logits);
                    *reinterpret_cast<float2*>(lg + ar * kLStride + na) = make_float2(v[0], v[1]);
                    *reinterpret_cast<float2*>(lg + (ar + 8) * kLStride + na) = make_float2(v[2], v[3]);
                    if (two) {
                        *reinterpret_cast<float2*>(lg + ar * kLStride + nb) = make_float2(v[4], v[5]);
                        *reinterpret_cast<float2*>(lg + (ar + 8) * kLStride + nb) = make_float2(v[6], v[7]);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = a.act == 0 ? tanh_mufu(v[j]) : fmaxf(v[j], 0.0f);
                    if (!two) v[4] = v[5] = v[6] = v[7] = 0.0f;
                    uint4 hi, lo;
                    split_f16x2(v[0], v[1], hi.x, lo.x);
                    split_f16x2(v[2], v[3], hi.y, lo.y);
                    split_f16x2(v[4], v[5], hi.z, lo.z);
                    split_f16x2(v[6], v[7], hi.w, lo.w);
                    reinterpret_cast<uint4*>(smem + ((l & 1) ? S.hhi[1] : S.hhi[0]))[(mt * KTn + jw) * 32 + lane] = hi;
                    reinterpret_cast<uint4*>(smem + ((l & 1) ? S.hlo[1] : S.hlo[0]))[(mt * KTn + jw) * 32 + lane] = lo;
                }
            }
            __syncthreads();
        }
        // ---- PolicyApply: one thread per row (f32 softmax, the reference's draw and walk)
        if (rowt) {
            const float* lg = reinterpret_cast<const float*>(smem + S.logits) + t * kLStride;
            // static loop bounds (predicated on A <= 16): p[] stays in registers
            float p[16];
            float mx = lg[0];
#pragma unroll
            for (int c = 1; c < 16; ++c)
                if (c < A) mx = fmaxf(mx, lg[c]);
            float den = 0.0f;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                p[c] = c < A ? __expf(lg[c] - mx) : 0.0f;
                den += p[c];
            }
            const float rden = 1.0f / den;
            double cum = 0.0;
            int chosen = A - 1;
            bool found = false;
#pragma unroll
            for (int c = 0; c < 16; ++c) {
                p[c] *= rden;
                if (c < A && !found) {
                    cum = __dadd_rn(cum, static_cast<double>(p[c]));
                    if (u < cum) {
                        chosen = c;
                        found = true;
                    }
                }
            }
            float pch = 0.0f;  // p[chosen]
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c == chosen) pch = p[c];
            acts[t] = chosen;
            const int64_t row = static_cast<int64_t>(ra) * E + re;
            a.actions[step * R + row] = chosen;
            a.logp[step * R + row] = __logf(fmaxf(pch, 1e-30f));
        }
        __syncthreads();
        // ---- EnvStep (envs.cpp:111-150; absorbing after done, interp.cpp:239-245): each row
        // thread moves its own agent, then scores it against the moved positions; the env thread
        // adds the agents' rewards in agent order and advances done / the step counter
        const bool live_row = rowt && !dns[rle];
        if (live_row) {  // moves (envs.cpp:114-126)
            double dx = 0.0, dy = 0.0;
            switch (acts[t]) {
                case 1: dx = 0.1; break;
                case 2: dx = -0.1; break;
                case 3: dy = 0.1; break;
                case 4: dy = -0.1; break;
                default: break;
            }
            sts[(2 * ra) * EPC + rle] = __dadd_rn(sts[(2 * ra) * EPC + rle], dx);
            sts[(2 * ra + 1) * EPC + rle] = __dadd_rn(sts[(2 * ra + 1) * EPC + rle], dy);
        }
        __syncthreads();
        if (rowt) {  // rewards (envs.cpp:128-144)
            double r = 0.0;
            if (live_row) {
                const double xa = sts[(2 * ra) * EPC + rle], ya = sts[(2 * ra + 1) * EPC + rle];
                double best = 1e18;
                for (int lm = 0; lm < n; ++lm) {
                    const double dx = __dsub_rn(sts[(2 * n + 2 * lm) * EPC + rle], xa);
                    const double dy = __dsub_rn(sts[(2 * n + 2 * lm + 1) * EPC + rle], ya);
                    const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
                    best = dist < best ? dist : best;
                }
                r = -best;
                for (int b = 0; b < n; ++b) {
                    if (b == ra) continue;
                    const double dx = __dsub_rn(sts[(2 * b) * EPC + rle], xa);
                    const double dy = __dsub_rn(sts[(2 * b + 1) * EPC + rle], ya);
                    if (__dsqrt_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy))) < 0.1) r = __dsub_rn(r, 0.5);
                }
            }
            rews[t] = r;
            a.reward[step * R + static_cast<int64_t>(ra) * E + re] = static_cast<float>(r);
        }
        __syncthreads();
        if (envt) {
            const int64_t e = e0 + t;
            double total = 0.0;
            bool d = true;
            if (!done) {
                for (int ag = 0; ag < n; ++ag) total = __dadd_rn(total, rews[ag * EPC + t]);
                d = a.env.max_steps > 0 && stepc + 1 >= a.env.max_steps;
                stepc += 1;
            }
            done = d;
            dns[t] = d ? 1 : 0;
            a.reward_d[step * E + e] = total;
            for (int ag = 0; ag < n; ++ag) a.done_f[step * R + static_cast<int64_t>(ag) * E + e] = d ? 1.0f : 0.0f;
        }
        __syncthreads();
        if (rowt) emit(step + 1);
        __syncthreads();
    }
    if (envt) {
        for (int i = 0; i < 4 * n; ++i) a.est[i * E + e0 + t] = sts[i * EPC + t];
        a.done[e0 + t] = done ? 1 : 0;
        a.stepc[e0 + t] = stepc;
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

namespace flw {
namespace {
inline int mappo_epc(int n) { return n <= 8 ? 16 : 8; }
}  // namespace

bool fast_rollout_mappo_ok(const FastRolloutArgs& a) {
    const int n = a.env.n_agents;
    if (a.env.kind != 2 || n < 1 || n > 16 || a.A > 16 || a.dims[0] > 64) return false;
    for (int l = 1; l < a.L; ++l)
        if (a.dims[l] > 64) return false;
    return mappo_carve(a, mappo_epc(n)).total <= 227u * 1024u;
}

void fast_rollout_mappo(cudaStream_t s, const DeviceCtx* ctx, const FastRolloutArgs& a) {
    const int epc = mappo_epc(a.env.n_agents);
    const size_t smem = mappo_carve(a, epc).total;
    const unsigned grid = static_cast<unsigned>((a.E + epc - 1) / epc);
    if (epc == 16) {
        FLW_CUDA(cudaFuncSetAttribute(k_rollout_mappo_fast<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k_rollout_mappo_fast<16><<<grid, 256, smem, s>>>(ctx, a);
    } else {
        FLW_CUDA(cudaFuncSetAttribute(k_rollout_mappo_fast<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
        k_rollout_mappo_fast<8><<<grid, 256, smem, s>>>(ctx, a);
    }
}

}  // namespace flw
