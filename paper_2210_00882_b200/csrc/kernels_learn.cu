// Fast-numerics learn phase, warp-specialised: one PPO/A3C train iteration of one MLP, fused
// per 128-row tile on the 5th-gen tensor cores (forward -> loss -> backward -> dW in TMEM).
//
// Every stage of a tile is a dependency chain (MMA -> TMEM load -> activation -> shared store ->
// proxy fence -> hand-off -> next MMA), so one tile per SM leaves the tensor pipe idle most of
// the time. Each CTA (one per SM, persistent over its tiles) keeps several tiles in flight:
//
//   warps [4g, 4g + 4)   epilogue group g (g < kGroups: 3 in the learn modes, 4 in the values
//                        pass): tile rows = TMEM lanes, one full row per thread
//   warp 4 kGroups       MMA producer 0 (even groups)   - one elected lane issues each
//   warp 4 kGroups + 1   loader (every TMA bulk copy: the forward's activation-tile stores,
//                        the backward's reloads)
//   warp 4 kGroups + 2   MMA producer 1 (odd groups)
//   warp 4 kGroups + 3   idle (learn modes: completes the warpgroup for setmaxnreg, which moves
//                        registers from these warps to the epilogue warps)
//
// Shared memory holds the bf16 weight image, per group a 2-slot activation ring (slot 1 also
// holds the input tile X) and one dZ slot, the bias rows and per-warp bias-gradient
// accumulators. The forward streams every hidden tile not kept resident out to global scratch
// and the backward streams it back one stage ahead. The critic learn pass skips its forward:
// its activations were saved by the values pass (same parameters) and are streamed from there.
//
// TMEM (512 columns): Z/dH accumulator of group g at columns [64g, 64g+64) (M=128); dW_l
// accumulators (M=64, half-sub-partition layout) of the layer pair (2j, 2j+1) after them, lane
// offsets 0 / 16 - shared by the groups and both producers, accumulated across all tiles in the
// single-issuer order (tile round, group) through the per-layer token dwtok: deterministic.
//
// Stage protocol per group: the producer waits epi_done[g] (all 4 epilogue warps stored their
// operand tile and fenced it to the async proxy), issues the stage's MMAs and commits to
// mma_done[g]; the epilogue waits mma_done[g], reads the accumulator, writes the next operand.
// A backward stage commits twice: dH_m to mma_done[g] (the epilogue starts on it) and dW_m, which
// still reads dZ_m from the dz slot, to dw_done[g]; the epilogue waits dw_done[g] just before it
// overwrites that slot with dZ_{m-1} (the next tile's first stores wait the last one).
#include <cuda_runtime.h>

// MODE 0 instantiations end each tile with `continue` before the learn-only stages
#pragma nv_diag_suppress 128

#include "common.cuh"
#include "fast.cuh"
#include "umma.cuh"

namespace flw {

namespace {

constexpr int kRows = 128;
constexpr int kMaxW = 64;
// tiles in flight per CTA (one epilogue group of 4 warps each): 3 in the learn modes (TMEM /
// shared memory hold their dZ slots and dW accumulators), 4 in the values pass (forward only)
__host__ __device__ constexpr int groups_for(int mode) { return mode == 0 ? 4 : 3; }
constexpr int kGroupsMax = 4;
constexpr int kGroups = groups_for(1);
// + two MMA producers (groups split by parity) + loader
// (learn modes: + one idle warp, so the non-epilogue warps form a whole warpgroup for setmaxnreg)
__host__ __device__ constexpr int threads_for(int mode) { return 32 * (4 * groups_for(mode) + (mode != 0 ? 4 : 3)); }
// learn modes: registers per thread after the role split (3 x 128 x 152 + 128 x 56 = 65536): the
// epilogue warps hold a row's accumulators, activations and loss inputs; the producers and the
// loader only issue
constexpr int kRegEpi = 152, kRegSide = 56;
constexpr uint32_t kSlot = kRows * kMaxW * 2;  // one 128 x 64 bf16 tile
constexpr int kXPre = 18;                      // input columns prefetched in registers (9 packed regs)
#ifndef FLW_TANH_MUFU_PAIRS
#define FLW_TANH_MUFU_PAIRS 4
#endif
constexpr int kMufuPairs = FLW_TANH_MUFU_PAIRS;  // of each 8-column chunk's 4 pairs: MUFU, rest poly

struct Carve {
    uint32_t wt[kMaxLayers], wbytes;
    uint32_t ring[kGroupsMax][2], dz[kGroupsMax];  // ring slot 1 also holds the input tile X
    uint32_t bias, dbacc, loss, total;
    uint32_t hoff[kMaxLayers + 1], hbytes;  // saved tile images: hoff[k + 1] = H_k, hoff[0] = X
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Carve carve_learn(const FastNet& n, int groups, bool learn) {
    Carve c{};
    uint32_t off = 0;
    for (int l = 0; l < n.L; ++l) {  // identical to the weight image built by k_build_wimg
        c.wt[l] = off;
        off = align_up(off + static_cast<uint32_t>(n.dout[l] * n.din[l] * 2), 128);
    }
    c.wbytes = off;
    off = align_up(off, 1024);
    for (int g = 0; g < groups; ++g) {
        for (int s = 0; s < 2; ++s) {
            c.ring[g][s] = off;
            off += kSlot;
        }
        if (learn) {
            c.dz[g] = off;
            off += kSlot;
        }
    }
    c.bias = off;
    off += kMaxLayers * kMaxW * 4;
    c.dbacc = off;
    if (learn) off += 4 * groups * kMaxLayers * kMaxW * 4;
    c.loss = off;
    off += 4 * groups * 3 * 4;
    c.total = off + 2048;  // slack: M=64 MN-major reads of narrow tiles run past their end
    uint32_t h = static_cast<uint32_t>(kRows * n.din[0] * 2);  // X first
    c.hoff[0] = 0;
    for (int l = 0; l + 1 < n.L; ++l) {
        c.hoff[l + 1] = h;
        h += static_cast<uint32_t>(kRows * n.dout[l] * 2);
    }
    c.hbytes = h;
    return c;
}

// Marks a value warp-uniform for ptxas (a lane-0 broadcast): descriptors and TMEM addresses built
// from such values stay in uniform registers, so each tcgen05.mma issues without per-operand
// R2UR.BROADCAST moves.
__device__ __forceinline__ uint32_t uni(uint32_t x) { return __shfl_sync(0xffffffffu, x, 0); }
__device__ __forceinline__ int uni(int x) { return __shfl_sync(0xffffffffu, x, 0); }

// Monotonic shared-memory hand-off counters (the loader may trail the epilogue by several
// stages, which a parity-tracked mbarrier cannot tell apart).
__device__ __forceinline__ void cnt_add_release(uint32_t* c) {
    asm volatile("red.release.cta.shared::cta.add.u32 [%0], 1;\n" ::"r"(umma::smem_u32(c)) : "memory");
}
__device__ __forceinline__ uint32_t cnt_acquire(const uint32_t* c) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];\n" : "=r"(v) : "r"(umma::smem_u32(c)) : "memory");
    return v;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(umma::smem_u32(bar)) : "memory");
}


__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// tanh on the FMA pipe (packed f32x2): odd polynomial of degree 17 on [-4, 4], saturated beyond;
// max abs error 1.7e-3 (below bf16 resolution near 1). Half of each 8-column chunk uses it, the
// other half MUFU.TANH, so the two pipes share the activation work.
__device__ __forceinline__ float2 tanh_poly2(float2 x) {
    x.x = fminf(fmaxf(x.x, -4.0f), 4.0f);
    x.y = fminf(fmaxf(x.y, -4.0f), 4.0f);
    const float2 t = __fmul2_rn(x, x);
    float2 p = make_float2(1.0064061584103001e-08f, 1.0064061584103001e-08f);
    p = __ffma2_rn(p, t, make_float2(-7.318681696233398e-07f, -7.318681696233398e-07f));
    p = __ffma2_rn(p, t, make_float2(2.24064351641573e-05f, 2.24064351641573e-05f));
    p = __ffma2_rn(p, t, make_float2(-0.00037694742786698043f, -0.00037694742786698043f));
    p = __ffma2_rn(p, t, make_float2(0.0038315874990075827f, 0.0038315874990075827f));
    p = __ffma2_rn(p, t, make_float2(-0.024628829210996628f, -0.024628829210996628f));
    p = __ffma2_rn(p, t, make_float2(0.10449711978435516f, 0.10449711978435516f));
    p = __ffma2_rn(p, t, make_float2(-0.3220818042755127f, -0.3220818042755127f));
    p = __ffma2_rn(p, t, make_float2(1.0f, 1.0f));
    return __fmul2_rn(p, x);
}


__device__ __forceinline__ void bulk_load(uint8_t* dst, const uint8_t* src, uint32_t bytes, uint64_t* bar) {
    umma::mbar_expect_tx(bar, bytes);
    for (uint32_t o = 0; o < bytes; o += 16384u) umma::bulk_g2s(dst + o, src + o, min(16384u, bytes - o), bar);
}


// Column sums over the warp's 32 rows of a 32-wide row slice held one row per lane: a
// reduce-scatter butterfly (31 shuffles); lane l ends with the sum of column l.
__device__ __forceinline__ float warp_colsum32(float* v, int lane) {
#pragma unroll
    for (int w = 16, off = 16; off > 0; w >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (i < w) {
                const float keep = up ? v[i + w] : v[i];
                const float send = up ? v[i] : v[i + w];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
    }
    return v[0];
}

// Column sums of an (at most) 8-wide row slice: three reduce-scatter levels (4 + 2 + 1
// shuffles) leave column (lane >> 2) & 7 summed over 8 lanes, two all-reduce levels finish it;
// every lane of the quad (lane >> 2) holds that column's sum.
__device__ __forceinline__ float warp_colsum8(float* v, int lane) {
#pragma unroll
    for (int w = 4, off = 16; off >= 4; w >>= 1, off >>= 1) {
        const bool up = (lane & off) != 0;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < w) {
                const float keep = up ? v[i + w] : v[i];
                const float send = up ? v[i] : v[i + w];
                v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
    }
    float s = v[0];
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    return s;
}

// acc + x for a bf16 x, rounded once to f32 (mixed-precision add: the bf16 half is read in place)
__device__ __forceinline__ float add_f32_bf16(float acc, uint16_t x) {
    asm("add.rn.f32.bf16 %0, %1, %0;" : "+f"(acc) : "h"(x));
    return acc;
}

// Column sums of the 32 rows [32 q, 32 q + 32) of a bf16 operand tile in shared memory (core-
// matrix layout, width C <= 64), added to acc[0, C): lane (k = lane & 7, s = lane >> 3) sums
// the 8-column chunk k over the 8 rows of core block 4q + s, reading them in the order rotated
// by k (the eight chunks of one read hit disjoint banks), then a two-level reduce-scatter over
// s (6 shuffles) leaves columns 8k + 4 s0 + 2 s1 + {0, 1} on the lane. Fixed order throughout.
__device__ __forceinline__ void warp_colsum_tile(const uint8_t* tile, int C, int q, int lane, float* acc) {
    const int k = lane & 7, s = lane >> 3;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.0f;
    if (8 * k < C) {
        const uint8_t* base = tile + (4 * q + s) * (C * 16) + k * 128;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint4 w = *reinterpret_cast<const uint4*>(base + ((i + k) & 7) * 16);
            const uint32_t p[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {  // f32 += bf16 (FHADD.BF16: no unpacking; exact widening)
                v[2 * j] = add_f32_bf16(v[2 * j], static_cast<uint16_t>(p[j] & 0xFFFFu));
                v[2 * j + 1] = add_f32_bf16(v[2 * j + 1], static_cast<uint16_t>(p[j] >> 16));
            }
        }
    }
    const bool up8 = (lane & 8) != 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float keep = up8 ? v[4 + i] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, up8 ? v[i] : v[4 + i], 8);
    }
    const bool up16 = (lane & 16) != 0;
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const float keep = up16 ? v[2 + i] : v[i];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, up16 ? v[i] : v[2 + i], 16);
    }
    if (8 * k < C) {
        float2* a2 = reinterpret_cast<float2*>(acc + 8 * k + (up8 ? 4 : 0) + (up16 ? 2 : 0));
        const float2 o = *a2;
        *a2 = make_float2(o.x + v[0], o.y + v[1]);
    }
}

// MODE 0: values pass (critic forward, saves activations); 1: learn (forward + backward);
// 2: learn reusing the values pass's activations (backward only). ACT 0: tanh, 1: relu.
// Compile-time modes keep each instantiation's code small (the stage loops are instruction-
// cache sensitive) and branch-free per activation chunk.
template <int MODE, int ACT, int NA>  // NA: output columns held by the loss epilogue (8 or 16)
__global__ void __launch_bounds__(threads_for(MODE), 1) k_learn(FastLearnArgs a, const __grid_constant__ Carve C) {
    constexpr int kGroups = groups_for(MODE);
    constexpr int kEpiWarps = 4 * kGroups;
    constexpr int kThreads = threads_for(MODE);
#ifndef FLW_LEARN_ZPRE  // forward epilogue: one TMEM round trip for all 64 columns (A/B: no gain,
#define FLW_LEARN_ZPRE 0  // values pass 0.1445 -> 0.1457 ms per episode)
#endif
    constexpr bool kZPre = FLW_LEARN_ZPRE;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mma_done[kGroups], dw_done[kGroups], epi_done[kGroups], ldbar[kGroups][2], wbar, zbar;
    __shared__ uint32_t tslot;
    __shared__ uint32_t dwtok[kMaxLayers];  // dW_l MMAs issued so far, in (tile round, group) order
    __shared__ uint32_t epi_cnt[kGroups];  // epilogue hand-offs per group (4 per stage), for the loader
    __shared__ uint32_t rd_cnt[kGroups];   // loader: bulk stores whose smem read completed (producer)
    __shared__ uint32_t xf_cnt[kGroups];   // loader, values pass: last saved tile read (epilogue)
    __shared__ double s_adv[2];            // advantage {mean, sd} (one unit: uniform over the rows)
    __shared__ int s_adv_on;
#ifdef FLW_LEARN_TRACE
    __shared__ long long tr_p[4][64], tr_e[3][64], tr_f[5][16], tr_b[4][32], tr_l[6][8];
    int np_ev = 0, ne_ev = 0, nf_ev = 0, nb_ev = 0, nl_ev = 0;
#endif
    const FastNet& n = a.net;
    const int t = threadIdx.x, w = uni(static_cast<int>(t >> 5)), lane = t & 31;
    const int L = n.L;
    const int64_t ntiles = (a.rows + kRows - 1) / kRows;
    const int G = gridDim.x;
    constexpr bool learn = MODE != 0;
    constexpr bool reuse = MODE == 2;  // critic: forward skipped, activations streamed in
    const bool fwd = !reuse;
    const int nfwd = fwd ? L : 0;
    const bool dx = learn && a.dx_out;  // also dZ wrt the net input (one extra stage per tile)
    const int njobs = learn ? nfwd + L : L;
    float* bias = reinterpret_cast<float*>(smem + C.bias);
    float* dbacc = reinterpret_cast<float*>(smem + C.dbacc);
    // H_k (k = -1: the input tile X) lives in ring slot k & 1; the last two the forward wrote
    // stay resident there (never reloaded)
    auto resident = [&](int k) { return fwd && (k == L - 2 || k == L - 3); };
    auto hwidth = [&](int k) { return k < 0 ? n.din[0] : n.dout[k]; };
    // where the forward saves H_k of a tile (k = -1: X): this group's scratch (learn, the tiles
    // the backward does not keep resident) or the values pass's save area; null: not saved
    auto save_dst = [&](int g, int64_t tile, int k) -> uint8_t* {
        if (learn) return resident(k) ? nullptr : a.hscratch + static_cast<size_t>(kGroups * blockIdx.x + g) * C.hbytes;
        return (a.hsave && tile < a.save_tiles) ? a.hsave + static_cast<size_t>(tile) * C.hbytes : nullptr;
    };

    // ---- setup
    if (t == 0) {
        for (int g = 0; g < kGroups; ++g) {
            umma::mbar_init(&mma_done[g], 1);
            umma::mbar_init(&dw_done[g], 1);
            umma::mbar_init(&epi_done[g], 4);
            umma::mbar_init(&ldbar[g][0], 1);
            umma::mbar_init(&ldbar[g][1], 1);

        }
        umma::mbar_init(&wbar, 1);
        umma::mbar_init(&zbar, 1);
        for (int g = 0; g < kGroups; ++g) epi_cnt[g] = rd_cnt[g] = xf_cnt[g] = 0;
        for (int l = 0; l < kMaxLayers; ++l) dwtok[l] = 0;
        umma::fence_barrier_init();
    }
    if (learn)
        for (int i = t; i < kEpiWarps * kMaxLayers * kMaxW / 4; i += kThreads)
            reinterpret_cast<float4*>(dbacc)[i] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
    if (learn) {  // dz slot of group 0 zeroed: the operand of the dW accumulators' zero-init MMAs
        for (uint32_t i = t; i < kSlot / 16; i += kThreads)
            reinterpret_cast<uint4*>(smem + C.dz[0])[i] = make_uint4(0u, 0u, 0u, 0u);
        umma::fence_async_smem();
    }
    if (w == 0) umma::tmem_alloc<512>(&tslot);
    // programmatic dependent launch (a.pdl): the setup above overlaps the update kernel before
    // this one; the weight image and the biases are that kernel's output
    if (a.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    if (t == 0) {
        bulk_load(smem, reinterpret_cast<const uint8_t*>(a.wimg), C.wbytes, &wbar);
        s_adv_on = a.adv_stats && !a.rep_of_env;  // (the GAE's output: possibly the kernel before)
        s_adv[0] = s_adv_on ? a.adv_stats[0] : 0.0;
        s_adv[1] = s_adv_on ? a.adv_stats[1] : 0.0;
    }
    for (int i = t; i < L * kMaxW; i += kThreads) {  // one global load per thread, all in flight
        const int l = i / kMaxW, o = i % kMaxW;
        bias[i] = o < n.rout[l] ? a.params[n.boff[l] + o] : 0.0f;
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = uni(tslot);
    const uint32_t sbase = umma::smem_u32(smem);

    // learn modes: the register file is rebalanced between the roles (per warpgroup: the
    // producers, the loader and the idle warp form the last one)
    auto regs_side = [&]() {
        if constexpr (MODE != 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegSide));
    };
    if (w == kEpiWarps || w == kEpiWarps + 2) {
        regs_side();
        // ================================================================ producer (whole warp)
        // The warp runs the issue loop converged (warp-uniform control flow and operands); one
        // elected lane issues each tcgen05.mma / commit / bulk copy (umma::mma_bf16_warp).
        {
            // two producer warps: groups of parity `pidx` each; the dW accumulators are shared,
            // so producer 0 zeroes them with one accumulate=0 MMA per layer on a zero operand
            // before either producer issues a stage, and every dW MMA accumulates
            const int pidx = w == kEpiWarps ? 0 : 1;
            umma::mbar_wait(&wbar, 0);
            // per-producer state of its own groups g = pidx + 2 gi, indexed by the compile-time gi
            // (runtime-indexed arrays would live in local memory): hand-off phases, the ldbar
            // phases as a bit mask (bit s: slot s), bulk-store reads required before a forward
            constexpr int kMine = (kGroups + 1) / 2;
            uint32_t ph_epi[kMine] = {}, ph_ld[kMine] = {}, need_rd[kMine] = {};
            auto dw_tmem = [&](int l) {
                return tmem + 64u * kGroups + 64u * static_cast<uint32_t>(l >> 1) + ((l & 1) ? (16u << 16) : 0u);
            };
            auto hsrc = [&](int g, int64_t tile) -> uint8_t* {
                return reuse ? a.hsave + static_cast<size_t>(tile) * C.hbytes
                             : a.hscratch + static_cast<size_t>(kGroups * blockIdx.x + g) * C.hbytes;
            };
            auto issue_dw = [&](int g, int l, uint32_t hin) {  // dW_l += H_{l-1}^T dZ_l  (M = din_l)
                const int di = n.din[l], dout = n.dout[l];
                const uint32_t dzt = uni(sbase + C.dz[g]);
                const uint32_t id = umma::idesc_bf16(64, dout, true, true);
                for (int kb = 0; kb < kRows / 16; ++kb)  // accumulators zeroed once below
                    umma::mma_bf16_warp(dw_tmem(l), umma::desc_mnmajor(hin, di, kb), umma::desc_mnmajor(dzt, dout, kb),
                                        id, true);
            };
            if (learn) {
                if (pidx == 0) {
                    const uint32_t zs = uni(sbase + C.dz[0]);
                    for (int l = 0; l < L; ++l)
                        umma::mma_bf16_warp(dw_tmem(l), umma::desc_mnmajor(zs, n.din[l], 0),
                                            umma::desc_mnmajor(zs, n.dout[l], 0),
                                            umma::idesc_bf16(64, n.dout[l], true, true), false);
                    umma::commit_warp(&zbar);
                }
                umma::mbar_wait(&zbar, 0);
                umma::fence_after_sync();
            }
            for (int64_t it = 0;; ++it) {
                // tiles are dealt to groups in ascending order: this producer's groups with a
                // tile this round are its first nmine (the groups past the end hold none)
                const int64_t t0 = it * kGroups * G + kGroups * static_cast<int64_t>(blockIdx.x);
                if (t0 + pidx >= ntiles) break;
                const int64_t avail = (ntiles - t0 - pidx + 1) / 2;
                const int nmine = avail < kMine ? static_cast<int>(avail) : kMine;
                for (int j = 0; j < njobs; ++j) {
#pragma unroll
                    for (int gi = 0; gi < kMine; ++gi) {
                        const int g = pidx + 2 * gi;
                        if (gi >= nmine || g >= kGroups) continue;
                        const int64_t tlg = t0 + g;
                        umma::mbar_wait(&epi_done[g], ph_epi[gi]);
                        ph_epi[gi] ^= 1;
#ifdef FLW_LEARN_TRACE
                        if (g == 0 && np_ev < 64) tr_p[0][np_ev] = clock64();
#endif
                        umma::fence_after_sync();
                        const uint32_t zt = tmem + 64u * static_cast<uint32_t>(g);
                        if (j < nfwd) {  // ---- forward layer l: Z = In_l W_l^T
                            const int l = j, di = n.din[l], dout = n.dout[l];
#ifdef FLW_LEARN_TRACE
                            if (g == 0 && np_ev < 64) tr_p[2][np_ev] = clock64();
#endif
                            // the epilogue of this job overwrites the slot of H_{l-2}: the loader's
                            // bulk store of it must have read the slot
                            if (l >= 1 && save_dst(g, tlg, l - 2)) {
                                ++need_rd[gi];
                                while (cnt_acquire(&rd_cnt[g]) < need_rd[gi]) __nanosleep(20);
                            }
                            const uint32_t in = uni(sbase + C.ring[g][(l - 1) & 1]);
                            const uint32_t wl = uni(sbase + C.wt[l]);
                            const uint32_t id = umma::idesc_bf16(128, dout, false, false);
                            for (int kb = 0; kb < di / 16; ++kb)
                                umma::mma_bf16_warp(zt, umma::desc_kmajor(in, di, kb),
                                               umma::desc_kmajor(wl, di, kb), id, kb > 0);
#ifdef FLW_LEARN_TRACE
                            if (g == 0 && np_ev < 64) tr_p[3][np_ev] = clock64();
#endif
                            umma::commit_warp(&mma_done[g]);
#ifdef FLW_LEARN_TRACE
                            if (g == 0 && np_ev < 64) tr_p[1][np_ev++] = clock64();
#endif
                        } else {  // ---- backward layer m: dH_m = dZ_m W_m and dW_m = H_{m-1}^T dZ_m
                            const int m = L - 1 - (j - nfwd);
                            // (the loader warp issues the activation tiles' TMA copies)
#ifdef FLW_LEARN_TRACE
                            if (g == 0 && np_ev < 64) tr_p[2][np_ev] = clock64();
#endif
                            const int sh = (m - 1) & 1;
                            const bool has_dh = m >= 1 || dx;
                            if (has_dh) {  // dH_m (m = 0: gradient wrt the input, dx mode)
                                const int di = n.din[m], dout = n.dout[m];
                                const uint32_t id = umma::idesc_bf16(128, di, false, true);
                                const uint32_t dzt = uni(sbase + C.dz[g]), wm = uni(sbase + C.wt[m]);
                                for (int kb = 0; kb < dout / 16; ++kb)
                                    umma::mma_bf16_warp(zt, umma::desc_kmajor(dzt, dout, kb),
                                                        umma::desc_mnmajor(wm, di, kb), id, kb > 0);
                                umma::commit_warp(&mma_done[g]);  // the epilogue starts on dH_m
                            }
                            if (!resident(m - 1)) {  // H_{m-1}: only dW_m reads it
                                umma::mbar_wait(&ldbar[g][sh], (ph_ld[gi] >> sh) & 1u);
                                ph_ld[gi] ^= 1u << sh;
                            }
                            // the shared dW_m accumulator takes its MMAs in the single-issuer order
                            // ((tile round, group) ascending), so the sums stay deterministic
                            const uint32_t want = static_cast<uint32_t>(it * kGroups + g);
                            while (cnt_acquire(&dwtok[m]) != want) {
                            }
                            umma::fence_after_sync();
                            issue_dw(g, m, uni(sbase + C.ring[g][sh]));
                            umma::fence_before_sync();
                            __syncwarp();
                            if (lane == 0) cnt_add_release(&dwtok[m]);
                            umma::commit_warp(has_dh ? &dw_done[g] : &mma_done[g]);
#ifdef FLW_LEARN_TRACE
                            if (g == 0 && np_ev < 64) tr_p[1][np_ev++] = clock64();
#endif
                        }
                    }
                }
            }
        }
    } else if (w == kEpiWarps + 1) {
        regs_side();
        // ================================================================ loader (learn modes)
        // The backward streams the activation tiles it does not keep resident back from global
        // memory (learn: this CTA's scratch, written by the producer's bulk stores during the
        // forward; learn-reuse: the values pass's save area). A second issuing warp follows the
        // producer's stage sequence (same epi_done hand-offs) and issues those TMA copies, so the
        // producer only issues MMAs (it waits the ldbar barriers). The copy into the slot of H_m
        // happens once stage m + 1's epilogue (its last reader, after stage m + 1's MMAs
        // completed) handed off; in learn mode the first one after the producer flushed its stores.
        {
            uint32_t seen[kGroups] = {};  // hand-offs consumed per group
            // the last bulk store whose smem read is not yet released (g * 2 + (values-pass last
            // tile ? 1 : 0), -1: none): released when the next store is issued (wait_group.read 1)
            // or before the loader would block waiting for a hand-off
            int pend = -1;
            auto release = [&](int e) { cnt_add_release((e & 1) ? &xf_cnt[e >> 1] : &rd_cnt[e >> 1]); };
            auto flush = [&]() {
                if (pend >= 0) {
                    if (lane == 0) {
                        umma::bulk_wait_read();
                        release(pend);
                    }
                    __syncwarp();
                    pend = -1;
                }
            };
            auto hsrc = [&](int g, int64_t tile) -> uint8_t* {
                return reuse ? a.hsave + static_cast<size_t>(tile) * C.hbytes
                             : a.hscratch + static_cast<size_t>(kGroups * blockIdx.x + g) * C.hbytes;
            };
            auto load_h = [&](int g, int64_t tile, int k) {  // H_k (k = -1: X) -> ring slot k & 1
                if (lane == 0) {
                    const uint32_t bytes = static_cast<uint32_t>(kRows * hwidth(k) * 2);
                    umma::mbar_expect_tx(&ldbar[g][k & 1], bytes);
                    umma::bulk_g2s_hint(smem + C.ring[g][k & 1], hsrc(g, tile) + C.hoff[k + 1], bytes,
                                        &ldbar[g][k & 1], umma::policy_evict_first());
                }
                __syncwarp();
            };
            for (int64_t it = 0;; ++it) {
                int64_t tl[kGroups];
                bool has[kGroups], any = false;
#pragma unroll
                for (int g = 0; g < kGroups; ++g) {
                    tl[g] = it * kGroups * G + kGroups * static_cast<int64_t>(blockIdx.x) + g;
                    has[g] = tl[g] < ntiles;
                    any = any || has[g];
                }
                if (!any) break;
                for (int j = 0; j < njobs; ++j) {
#pragma unroll
                    for (int g = 0; g < kGroups; ++g) {
                        if (!has[g]) continue;
                        ++seen[g];
                        if (cnt_acquire(&epi_cnt[g]) < 4u * seen[g]) {
                            flush();
                            while (cnt_acquire(&epi_cnt[g]) < 4u * seen[g]) __nanosleep(20);
                        }
                        if (j < nfwd) {  // forward job l: H_{l-1} (X for l = 0) is complete, save it
                            const int hk = j - 1;
                            uint8_t* gdst = save_dst(g, tl[g], hk);
                            if (gdst) {
                                if (lane == 0) {  // the critic learn re-reads the values pass's tiles
                                    umma::bulk_s2g_hint(gdst + C.hoff[hk + 1], smem + C.ring[g][hk & 1],
                                                        static_cast<uint32_t>(kRows * hwidth(hk) * 2),
                                                        learn ? umma::policy_evict_first() : umma::policy_evict_last());
                                    umma::bulk_commit();
                                    if (pend >= 0) {  // every older store has read its slot
                                        umma::bulk_wait_read1();
                                        release(pend);
                                    }
                                }
                                __syncwarp();
                                // values pass: the last saved tile shares its slot with the next
                                // tile's X, which the epilogue writes (not an MMA)
                                pend = 2 * g + (!learn && hk == L - 2 ? 1 : 0);
                            }
                            continue;
                        }
                        const int m = L - 1 - (j - nfwd);
                        if (j == nfwd && fwd) {  // this tile's stores are in global memory
                            flush();
                            if (lane == 0) umma::bulk_wait_all();
                            __syncwarp();
                            asm volatile("fence.proxy.async.global;\n" ::: "memory");
                        }
                        if (j == nfwd && !resident(m - 1)) load_h(g, tl[g], m - 1);
                        if (m - 2 >= -1 && !resident(m - 2)) load_h(g, tl[g], m - 2);
                    }
                }
            }
            flush();
            if (lane == 0) umma::bulk_wait_all();  // values pass: the saved tiles are written
            __syncwarp();
        }
    } else if (w < kEpiWarps) {
        if constexpr (MODE != 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegEpi));
        // ================================================================ epilogue groups
        // the dW zero-init MMAs read group 0's dz slot: no dZ store before they completed
        // (learn-reuse writes dZ_{L-1} before any MMA of its own)
        if (learn) umma::mbar_wait(&zbar, 0);
        const int g = w >> 2, q = w & 3;
        const int r = 32 * q + lane;  // tile row == TMEM lane
        const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
        const uint32_t zt = tmem + lane_base + 64u * static_cast<uint32_t>(g);
        uint32_t ph_mma = 0, ph_dw = 0, ph_ld = 0, need_xf = 0;  // ph_ld: bit s = phase of ldbar slot s
        float pl_acc = 0.0f, vl_acc = 0.0f, en_acc = 0.0f;
        float* mydb = dbacc + w * kMaxLayers * kMaxW;
        const int din0 = n.din[0];
        const bool xpre = a.in_cols <= kXPre;
        uint32_t xnext[kXPre / 2];  // next tile's input row, already packed to bf16 pairs
        auto fetch_x = [&](int64_t tile) {
            const int64_t rw = tile * kRows + r;
            const bool ok = tile < ntiles && rw < a.rows;
#pragma unroll
            for (int c = 0; c < kXPre; c += 2) {
                const float x0 = (ok && c < a.in_cols) ? a.X[rw * a.in_cols + c] : 0.0f;
                const float x1 = (ok && c + 1 < a.in_cols) ? a.X[rw * a.in_cols + c + 1] : 0.0f;
                xnext[c / 2] = umma::pack_bf16x2(x0, x1);
            }
        };
        auto signal = [&]() {  // operand tile stored: hand it to the producer
            // generic-proxy shared-memory writes (operand tiles) -> visible to the tensor core
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&epi_done[g]);
                cnt_add_release(&epi_cnt[g]);
            }
#ifdef FLW_LEARN_TRACE
            if (t == 0 && ne_ev > 0 && ne_ev <= 64) tr_e[2][ne_ev - 1] = clock64();
#endif
        };
        auto wait_mma = [&]() {
#ifdef FLW_LEARN_TRACE
            if (t == 0 && ne_ev < 64) tr_e[0][ne_ev] = clock64();
#endif
            umma::mbar_wait(&mma_done[g], ph_mma);
            ph_mma ^= 1;
            umma::fence_after_sync();
#ifdef FLW_LEARN_TRACE
            if (t == 0 && ne_ev < 64) tr_e[1][ne_ev++] = clock64();
#endif
        };
        auto wait_dw = [&]() {  // this group's last dW MMAs completed: the dz slot is free
            umma::mbar_wait(&dw_done[g], ph_dw);
            ph_dw ^= 1;
            umma::fence_after_sync();
        };
        // loads accumulator columns [c0, c0 + 32) of this thread's row (those below `width`)
        auto ld_acc32 = [&](float* v, int c0, int width) {
            umma::tmem_ld16(zt + c0, v);
            if (c0 + 16 < width) umma::tmem_ld16(zt + c0 + 16, v + 16);
            umma::tmem_ld_wait();
        };
        // db_layer[c0 + lane] += column sum of this warp's 32 rows (fixed order, no atomics)
        auto colsum32 = [&](float* v, int c0, int width, int layer) {
#pragma unroll
            for (int c = 0; c < 32; ++c)
                if (c0 + c >= width) v[c] = 0.0f;
            if (width - c0 <= 8) {  // the output layer (A or 1 columns)
                const float sum = warp_colsum8(v, lane);
                if ((lane & 3) == 0) mydb[layer * kMaxW + c0 + (lane >> 2)] += sum;
            } else {
                const float sum = warp_colsum32(v, lane);
                mydb[layer * kMaxW + c0 + lane] += sum;
            }
        };
        bool first = true;
        uint8_t* const xs = smem + C.ring[g][1];  // the input tile X lives in ring slot 1
        if (xpre && fwd) fetch_x(kGroups * static_cast<int64_t>(blockIdx.x) + g);
        for (int64_t tile = kGroups * static_cast<int64_t>(blockIdx.x) + g; tile < ntiles; tile += kGroups * G) {
            const int64_t row = tile * kRows + r;
            const bool valid = row < a.rows;
            // previous tile's last MMAs (dW_0) released X and dZ
            if (learn && !first) dx ? wait_dw() : wait_mma();
            if (!learn && !first && save_dst(g, tile - kGroups * G, L - 2)) {  // values pass: see the loader
                ++need_xf;
                while (cnt_acquire(&xf_cnt[g]) < need_xf) __nanosleep(20);
            }
            first = false;
            // ---- input tile (f32 -> bf16); learn-reuse: X comes from the values pass's save area
            if (!fwd) {
            } else if (!xpre) {
                for (int c0 = 0; c0 < din0; c0 += 8) {
                    float u[8];
                    for (int j = 0; j < 8; ++j) {
                        const int c = c0 + j;
                        u[j] = (valid && c < a.in_cols) ? a.X[row * a.in_cols + c] : 0.0f;
                    }
                    umma::st_row8(xs, din0, r, c0, u);
                }
            } else {
#pragma unroll
                for (int c0 = 0; c0 < 24; c0 += 8)  // 8-column chunks; pairs beyond kXPre are zero
                    if (c0 < din0) {
                        uint32_t q4[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) q4[i] = c0 / 2 + i < kXPre / 2 ? xnext[c0 / 2 + i] : 0u;
                        *reinterpret_cast<uint4*>(xs + umma::tile_offset(r, c0, din0)) =
                            make_uint4(q4[0], q4[1], q4[2], q4[3]);
                    }
                for (int c0 = 24; c0 < din0; c0 += 8)  // padded input columns: zeros
                    *reinterpret_cast<uint4*>(xs + umma::tile_offset(r, c0, din0)) = make_uint4(0u, 0u, 0u, 0u);
                fetch_x(tile + kGroups * G);
            }
            int act_r = 0, rep_r = 0;
            float lpo_r = 0.0f, adv_r = 0.0f, ret_r = 0.0f, val_r = 0.0f, inv_n_r = 0.0f;
            // the loss epilogue's per-row inputs: issued two forward stages ahead of their use
            // (not at the tile start), so they are neither held across the whole forward nor
            // waited for at the loss stage
            auto load_rows = [&]() {
                if (learn && valid) {
                    if (a.kind != kNetPolicyPpo) ret_r = a.ret[row];
                    if (a.kind != kNetCritic) act_r = a.actions[row];
                    if (a.kind == kNetPolicyPpo) {
                        lpo_r = a.logp_old[row];
                        adv_r = a.adv[row];
                    }
                    if (a.kind == kNetPolicyA3c || reuse) val_r = a.values_in[row];
                    if (a.rep_of_env) rep_r = a.rep_of_env[row % a.rep_E];
                }
            };
            // the row's loss weight and normalised advantage, computed while the last forward
            // MMA runs (the statistics' loads and the double division are off the loss stage)
            auto prep_rows = [&]() {
                if (!(learn && valid)) return;
                inv_n_r = static_cast<float>(a.inv_n);
                double am = s_adv[0], asd = s_adv[1];
                bool norm = s_adv_on != 0;
                if (a.rep_of_env) {  // folded replicas: this row's unit weight and statistics
                    inv_n_r = a.rep_w[rep_r];
                    if (a.adv_stats) {
                        am = a.adv_stats[2 * rep_r];
                        asd = a.adv_stats[2 * rep_r + 1];
                        norm = true;
                    }
                }
                if (a.kind == kNetPolicyPpo && norm && !(asd < 1e-8))
                    adv_r = static_cast<float>((adv_r - am) / (asd + 1e-8));
            };
            if (!fwd) {
                load_rows();
                prep_rows();
            }
            float out[NA];
            if (fwd) {
                signal();  // X ready
                for (int l = 0; l < L; ++l) {
                    const int dout = n.dout[l];
                    if (l == (L > 2 ? L - 2 : 0)) load_rows();
                    if (l == L - 1) prep_rows();
                    wait_mma();
                    const float* bl = bias + l * kMaxW;
                    if (l + 1 < L) {
                        uint8_t* dst = smem + C.ring[g][l & 1];
                        // (the producer bulk-stores the finished tile for the backward / critic learn)
                        // 32 columns of H_l = act(Z + b); FULL: no per-chunk guards, so the
                        // compiler interleaves the four 8-column chains
                        auto half = [&]<bool FULL, bool LOADED>(int h0, float* zin) {
                            float zl[32];
                            float* z = LOADED ? zin : zl;
                            if constexpr (!LOADED) {
                                umma::tmem_ld16(zt + h0, zl);
                                if (FULL || h0 + 16 < dout) umma::tmem_ld16(zt + h0 + 16, zl + 16);
                                umma::tmem_ld_wait();
                            }
#pragma unroll
                            for (int c = 0; c < 32; c += 8) {
                                if (FULL || h0 + c < dout) {
                                    const float4 b0 = *reinterpret_cast<const float4*>(bl + h0 + c);
                                    const float4 b1 = *reinterpret_cast<const float4*>(bl + h0 + c + 4);
                                    const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
                                    uint32_t p[4];
#pragma unroll
                                    for (int i = 0; i < 4; ++i) {
                                        // bias add as one packed f32x2 add (same rounding as two)
                                        const float2 zz = __fadd2_rn(make_float2(z[c + 2 * i], z[c + 2 * i + 1]),
                                                                     make_float2(bb[2 * i], bb[2 * i + 1]));
                                        const float z0 = zz.x, z1 = zz.y;
                                        if constexpr (ACT != 0) {
                                            p[i] = umma::pack_bf16x2(fmaxf(z0, 0.0f), fmaxf(z1, 0.0f));
                                        } else if (i < kMufuPairs) {
                                            p[i] = umma::pack_bf16x2(tanh_fast(z0), tanh_fast(z1));
                                        } else {
                                            const float2 y2 = tanh_poly2(make_float2(z0, z1));
                                            p[i] = umma::pack_bf16x2(y2.x, y2.y);
                                        }
                                    }
                                    const uint32_t off = umma::tile_offset(r, h0 + c, dout);
                                    const uint4 v4 = make_uint4(p[0], p[1], p[2], p[3]);
                                    *reinterpret_cast<uint4*>(dst + off) = v4;
                                }
                            }
                        };
#ifdef FLW_LEARN_TRACE
                        const bool trf = learn && g == 0 && t == 0 && nf_ev < 16;
                        if (trf) tr_f[0][nf_ev] = clock64();
#endif
                        if (dout == kMaxW && kZPre) {
                            // all 64 accumulator columns in one TMEM round trip
                            float z0[32], z1[32];
                            umma::tmem_ld16(zt, z0);
                            umma::tmem_ld16(zt + 16, z0 + 16);
                            umma::tmem_ld16(zt + 32, z1);
                            umma::tmem_ld16(zt + 48, z1 + 16);
                            umma::tmem_ld_wait();
                            half.template operator()<true, true>(0, z0);
                            half.template operator()<true, true>(32, z1);
                        } else if (dout == kMaxW) {
                            half.template operator()<true, false>(0, nullptr);
#ifdef FLW_LEARN_TRACE
                            if (trf) tr_f[1][nf_ev] = clock64();
#endif
                            half.template operator()<true, false>(32, nullptr);
                        } else {
                            for (int h0 = 0; h0 < dout; h0 += 32) half.template operator()<false, false>(h0, nullptr);
                        }
#ifdef FLW_LEARN_TRACE
                        if (trf) tr_f[2][nf_ev] = clock64();
#endif
                        signal();  // H_l ready
#ifdef FLW_LEARN_TRACE
                        if (trf) tr_f[3][nf_ev] = clock64();
#endif
#ifdef FLW_LEARN_TRACE
                        if (trf) tr_f[4][nf_ev++] = clock64();
#endif
                    } else {
                        float z[32];
                        ld_acc32(z, 0, 16);
#pragma unroll
                        for (int j = 0; j < NA; ++j) out[j] = z[j] + bl[j];
                    }
                }
            } else {
                out[0] = val_r;
            }
            if (!learn) {  // values pass
                if (valid) {
                    if (a.split_rows >= 0 && row >= a.split_rows)
                        a.values_out2[row - a.split_rows] = out[0];
                    else
                        a.values_out[row] = out[0];
                }
                continue;
            }
            // ---- loss epilogue (rl.cpp:137-202 semantics, f32) -> dZ_{L-1}
#ifdef FLW_LEARN_TRACE
            const bool trl = g == 0 && t == 0 && nl_ev < 8;
            if (trl) tr_l[0][nl_ev] = clock64();
#endif
            // Static loop bounds only (predicated on the action count) and the probabilities
            // recomputed per use instead of held in arrays: out[] and dz[] stay in registers.
            {
                float dz[NA];  // output layer width <= NA (the loss epilogue owns the whole row)
#pragma unroll
                for (int j = 0; j < NA; ++j) dz[j] = 0.0f;
                if (valid) {
                    const float inv_n = inv_n_r;
                    if (a.kind == kNetCritic) {  // value MSE: dV = 2 c_v (V - R) / N
                        const float verr = out[0] - ret_r;
                        dz[0] = static_cast<float>(2.0 * a.value_coef) * inv_n * verr;
                        vl_acc += static_cast<float>(a.value_coef) * inv_n * verr * verr;
                    } else {  // policy: clipped surrogate (PPO) or A3C policy gradient, + entropy bonus
                        const int A = n.rout[L - 1];
                        float mx = out[0];
#pragma unroll
                        for (int j = 1; j < NA; ++j)
                            if (j < A) mx = fmaxf(mx, out[j]);
                        // the exponentials once (the MUFU pipe is shared with the other groups'
                        // tanh epilogues: every dependent MUFU stage here queues behind them)
                        float pr[NA], den = 0.0f;
#pragma unroll
                        for (int j = 0; j < NA; ++j) {
                            pr[j] = j < A ? __expf(out[j] - mx) : 0.0f;
                            den += pr[j];
                        }
                        const float lden = __logf(den), rden = __fdividef(1.0f, den);
#pragma unroll
                        for (int j = 0; j < NA; ++j) pr[j] *= rden;  // probabilities
#ifdef FLW_LEARN_TRACE
                        if (trl) tr_l[3][nl_ev] = clock64();
#endif
                        float H = 0.0f, lpa = 0.0f;
#pragma unroll
                        for (int j = 0; j < NA; ++j) {
                            if (j < A) {
                                const float lp = out[j] - mx - lden;
                                H -= pr[j] * lp;
                                if (j == act_r) lpa = lp;
                            }
                        }
                        float coef;
                        if (a.kind == kNetPolicyPpo) {
                            const float adv = adv_r;  // normalised by prep_rows
                            const float ratio = __expf(lpa - lpo_r);
                            const float clipped = fminf(fmaxf(ratio, 1.0f - a.clip_eps), 1.0f + a.clip_eps);
                            const float s1 = ratio * adv, s2 = clipped * adv;
                            pl_acc -= fminf(s1, s2) * inv_n;
                            coef = s1 <= s2 ? -inv_n * ratio * adv : 0.0f;
                        } else {  // A3C: advantage R - V (rl.cpp:188)
                            const float adv = ret_r - val_r;
                            pl_acc -= lpa * adv * inv_n;
                            coef = -inv_n * adv;
                        }
                        en_acc += H * inv_n;
#ifdef FLW_LEARN_TRACE
                        if (trl) tr_l[4][nl_ev] = clock64();
#endif
                        const float eci = static_cast<float>(a.entropy_coef) * inv_n;
#pragma unroll
                        for (int j = 0; j < NA; ++j) {
                            if (j < A) {
                                const float lp = out[j] - mx - lden, pj = pr[j];
                                dz[j] = coef * ((j == act_r ? 1.0f : 0.0f) - pj) + eci * pj * (lp + H);
                            }
                        }
                    }
                }
                const int wo = n.dout[L - 1];
                uint8_t* dst = smem + C.dz[g];
#pragma unroll
                for (int c0 = 0; c0 < 16; c0 += 8) {
                    if (c0 < wo) {
                        if (c0 < NA) {
                            // round to the bf16 operand first so db sums exactly what dW sees
#pragma unroll
                            for (int i = 0; i < 8; ++i) dz[c0 + i] = __bfloat162float(__float2bfloat16(dz[c0 + i]));
                            umma::st_row8(dst, wo, r, c0, dz + c0);
                        } else {  // padding columns of the output layer
                            *reinterpret_cast<uint4*>(dst + umma::tile_offset(r, c0, wo)) = make_uint4(0u, 0u, 0u, 0u);
                        }
                    }
                }
#ifdef FLW_LEARN_TRACE
                if (trl) tr_l[5][nl_ev] = clock64();
#endif
                signal();  // dZ_{L-1} ready
#ifdef FLW_LEARN_TRACE
                if (trl) tr_l[1][nl_ev] = clock64();
#endif
                // bias gradient of the output layer: columns >= rout are zero
                const int ro = n.rout[L - 1];
                if (ro <= 8) {
                    const float sum = warp_colsum8(dz, lane);
                    if ((lane & 3) == 0) mydb[(L - 1) * kMaxW + (lane >> 2)] += sum;
                } else {
                    float v32[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) v32[c] = c < NA ? dz[c] : 0.0f;
                    colsum32(v32, 0, wo, L - 1);
                }
            }
#ifdef FLW_LEARN_TRACE
            if (trl) tr_l[2][nl_ev++] = clock64();
#endif
            // ---- backward epilogues: dZ_{m-1} = dH_m * act'(H_{m-1})
            for (int m = L - 1; m >= 1; --m) {
                const int di = n.din[m];
                wait_mma();
                const int s = (m - 1) & 1;
                if (!resident(m - 1)) {
                    umma::mbar_wait(&ldbar[g][s], (ph_ld >> s) & 1u);
                    ph_ld ^= 1u << s;
                }
                const uint8_t* hs = smem + C.ring[g][s];
                uint8_t* dst = smem + C.dz[g];
#ifdef FLW_LEARN_TRACE
                const bool trb = g == 0 && t == 0 && nb_ev < 32;
                if (trb) tr_b[0][nb_ev] = clock64();
#endif
                auto half = [&]<bool FULL, int h0>() {
                    float gv[32];
                    umma::tmem_ld16(zt + h0, gv);
                    if (FULL || h0 + 16 < di) umma::tmem_ld16(zt + h0 + 16, gv + 16);
                    umma::tmem_ld_wait();
                    if (h0 == 0) wait_dw();  // dW_m has read dZ_m: the slot takes dZ_{m-1}
#pragma unroll
                    for (int c = 0; c < 32; c += 8) {
                        if (FULL || h0 + c < di) {
                            float y[8];
                            umma::ld_row8(hs, di, r, h0 + c, y);
                            uint32_t pk[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const float2 yy = make_float2(y[2 * i], y[2 * i + 1]);
                                const float2 gg = make_float2(gv[c + 2 * i], gv[c + 2 * i + 1]);
                                float2 d;
                                if constexpr (ACT == 0) {  // dZ = dH (1 - y^2), packed f32x2 on the FMA pipe
                                    const float2 om = __ffma2_rn(make_float2(-yy.x, -yy.y), yy, make_float2(1.0f, 1.0f));
                                    d = __fmul2_rn(gg, om);
                                } else {
                                    d = make_float2(yy.x > 0.0f ? gg.x : 0.0f, yy.y > 0.0f ? gg.y : 0.0f);
                                }
                                pk[i] = umma::pack_bf16x2(d.x, d.y);
                            }
                            *reinterpret_cast<uint4*>(dst + umma::tile_offset(r, h0 + c, di)) =
                                make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        }
                    }
                };
                if (di == kMaxW) {
                    half.template operator()<true, 0>();
#ifdef FLW_LEARN_TRACE
                    if (trb) tr_b[1][nb_ev] = clock64();
#endif
                    half.template operator()<true, 32>();
                } else {
                    half.template operator()<false, 0>();
                    if (32 < di) half.template operator()<false, 32>();
                }
                signal();  // dZ_{m-1} complete: hand it to the producer
#ifdef FLW_LEARN_TRACE
                if (trb) tr_b[2][nb_ev] = clock64();
#endif
                // bias gradient off the hand-off path: column sums of this warp's 32 rows of the
                // bf16 dZ_{m-1} just stored (exactly the operand dW sees), read back from the slot
                warp_colsum_tile(dst, di, q, lane, mydb + (m - 1) * kMaxW);
#ifdef FLW_LEARN_TRACE
                if (trb) tr_b[3][nb_ev++] = clock64();
#endif

            }
            if (!resident(-1) && !dx) ph_ld ^= 2u;  // X's reload (stage 0): consumed by the producer only
            if (dx) {  // dZ wrt the input pre-activation: dH_0 * act'(X), X = the input tile (bf16)
                wait_mma();
                if (!resident(-1)) {
                    umma::mbar_wait(&ldbar[g][1], (ph_ld >> 1) & 1u);
                    ph_ld ^= 2u;
                }
                const int di = n.din[0];
                for (int h0 = 0; h0 < di; h0 += 32) {
                    float gv[32];
                    ld_acc32(gv, h0, di);
#pragma unroll
                    for (int c = 0; c < 32; c += 8) {
                        if (h0 + c < di) {
                            float y[8];
                            umma::ld_row8(xs, di, r, h0 + c, y);
#pragma unroll
                            for (int i = 0; i < 8; ++i) {
                                const int col = h0 + c + i;
                                const float d = ACT == 0 ? gv[c + i] * (1.0f - y[i] * y[i])
                                                           : (y[i] > 0.0f ? gv[c + i] : 0.0f);
                                if (valid && col < a.in_cols) a.dx_out[row * a.in_cols + col] = d;
                            }
                        }
                    }
                }
            }
        }
        if (learn && !first) dx ? wait_dw() : wait_mma();  // the last tile's dW_0
        // ---- loss partials of this warp
        for (int off = 16; off > 0; off >>= 1) {
            pl_acc += __shfl_xor_sync(0xffffffffu, pl_acc, off);
            vl_acc += __shfl_xor_sync(0xffffffffu, vl_acc, off);
            en_acc += __shfl_xor_sync(0xffffffffu, en_acc, off);
        }
        if (lane == 0) {
            float* ls = reinterpret_cast<float*>(smem + C.loss);
            ls[w * 3 + 0] = pl_acc;
            ls[w * 3 + 1] = vl_acc;
            ls[w * 3 + 2] = en_acc;
        }
    } else {
        regs_side();  // the idle warp (learn modes)
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();

    // a programmatic dependent (the update kernel) may launch once every CTA is here: its
    // prologue overlaps this CTA's partial-slot store
    if constexpr (learn) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // ---- per-CTA partials: dW from TMEM, db and loss terms from shared memory (fixed order).
    // The slot is assembled in the (now idle) activation slots and leaves as one bulk copy: the
    // TMEM lane layout puts one dW row per lane, so direct stores would be 4-byte writes
    // strided by a row (partial-sector L2 writes, ~9% of the kernel in ncu r02e).
    const bool any = kGroups * static_cast<int64_t>(blockIdx.x) < ntiles;
    float* part = learn ? a.partials + static_cast<int64_t>(blockIdx.x) * a.part_stride : nullptr;
    const bool staged = learn && any && static_cast<uint64_t>(a.part_stride) * 4u <= C.bias - C.ring[0][0];
    float* stage = reinterpret_cast<float*>(smem + C.ring[0][0]);
    float* dst = staged ? stage : part;
    if (learn && w < kEpiWarps) {
        const int q = w & 3, half = w >> 2;
        const uint32_t lane_base = static_cast<uint32_t>(32 * q) << 16;
        for (int l = 0; l < L; ++l) {
            const int dout = n.dout[l], ri = n.rin[l], ro = n.rout[l];
            const int lo = (l & 1) ? 16 : 0;
            const uint32_t col = 64u * kGroups + 64u * static_cast<uint32_t>(l >> 1);
            const int64_t base = n.woff[l] - n.woff[0];
            const bool vec = staged && ((base | ro) & 3) == 0;
            for (int c0 = 16 * half; c0 < dout; c0 += 16 * kGroups) {
                float v[16];
                umma::tmem_ld16(tmem + lane_base + col + c0, v);
                umma::tmem_ld_wait();
                const int mrow = lane - lo;  // dW row (input index) held by this lane
                if (any && mrow >= 0 && mrow < 16) {
                    const int i = mrow + 16 * q;
                    if (i < ri) {
                        float* rowp = dst + base + static_cast<int64_t>(i) * ro + c0;
                        if (vec) {
#pragma unroll
                            for (int j = 0; j < 16; j += 4)
                                if (c0 + j < ro)
                                    *reinterpret_cast<float4*>(rowp + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 16; ++j)
                                if (c0 + j < ro) rowp[j] = v[j];
                        }
                    }
                }
            }
            for (int o = t; o < ro; o += 32 * kEpiWarps) {
                float s = 0.0f;
                for (int k = 0; k < kEpiWarps; ++k) s += dbacc[(k * kMaxLayers + l) * kMaxW + o];
                dst[n.boff[l] - n.woff[0] + o] = s;
            }
        }
        if (t < 3) {
            const float* ls = reinterpret_cast<const float*>(smem + C.loss);
            float s = 0.0f;
            for (int k = 0; k < kEpiWarps; ++k) s += ls[k * 3 + t];
            a.loss_partials[blockIdx.x * 3 + t] = s;
        }
        if (!any)
            for (int64_t i = t; i < a.part_stride; i += 32 * kEpiWarps) part[i] = 0.0f;
    }
    if (staged) {
        umma::fence_async_smem();  // the generic stores above -> the bulk copy's async proxy
        __syncthreads();
        const uint64_t bytes = static_cast<uint64_t>(a.part_stride) * 4u;
        if ((reinterpret_cast<uintptr_t>(part) & 15u) == 0 && (bytes & 15u) == 0) {
            if (t == 0) {
                umma::bulk_s2g(part, stage, static_cast<uint32_t>(bytes));
                umma::bulk_commit();
                umma::bulk_wait_all();
            }
        } else {
            for (int64_t i = t; i < a.part_stride; i += kThreads) part[i] = stage[i];
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_free<512>(tmem);
#ifdef FLW_LEARN_TRACE
    if (blockIdx.x == 0 && t == 0 && MODE != 0) {
        const long long t0 = tr_p[0][0];
        for (int i = 0; i < ne_ev; ++i)
            printf("E%d %2d wait %7lld got %7lld signal %7lld\n", MODE, i, tr_e[0][i] - t0, tr_e[1][i] - t0, tr_e[2][i] - t0);
        for (int i = 0; i < nb_ev; ++i)
            printf("B %2d got %7lld half0 %7lld signaled %7lld end %7lld\n", i, tr_b[0][i] - t0, tr_b[1][i] - t0,
                   tr_b[2][i] - t0, tr_b[3][i] - t0);
        for (int i = 0; i < nl_ev; ++i)
            printf("L %2d start %7lld softmax %7lld coef %7lld stored %7lld signaled %7lld end %7lld\n", i, tr_l[0][i] - t0,
                   tr_l[3][i] - t0, tr_l[4][i] - t0, tr_l[5][i] - t0, tr_l[1][i] - t0, tr_l[2][i] - t0);
        for (int i = 0; i < nf_ev; ++i)
            printf("F %2d start %7lld half0 %7lld stores %7lld signaled %7lld bulk %7lld\n", i, tr_f[0][i] - t0,
                   tr_f[1][i] - t0, tr_f[2][i] - t0, tr_f[3][i] - t0, tr_f[4][i] - t0);
    }
    if (blockIdx.x == 0 && t == 32 * kEpiWarps && MODE != 0) {
        const long long t0 = tr_p[0][0];
        for (int i = 0; i < np_ev; ++i)
            printf("P%d %2d epi %7lld a %7lld b %7lld commit %7lld\n", MODE, i, tr_p[0][i] - t0, tr_p[2][i] - t0,
                   tr_p[3][i] - t0, tr_p[1][i] - t0);
    }
#endif
}

}  // namespace

size_t fast_learn_smem_bytes(const FastNet& n) { return carve_learn(n, kGroups, true).total; }
size_t fast_learn_scratch_bytes(const FastNet& n) { return carve_learn(n, kGroups, true).hbytes; }
int fast_learn_groups() { return kGroups; }
int fast_values_groups() { return groups_for(0); }

void fast_learn(cudaStream_t s, const FastLearnArgs& a, int grid) {
    const int mode = a.mode != 1 ? 0 : (a.hload && a.net.L > 1 ? 2 : 1);
    const Carve carve = carve_learn(a.net, groups_for(mode), mode != 0);  // smem offsets: a kernel argument
    const size_t smem = carve.total;
    if (smem > 227u * 1024u) throw Error(Errc::Config, "fast numerics: network too wide/deep for one SM's shared memory");
    auto go = [&](auto kern) {
        // per-device attribute: set on every launch (cheap, and legal inside stream capture)
        FLW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        if (!a.pdl) {
            kern<<<grid, threads_for(mode), smem, s>>>(a, carve);
            FLW_CUDA(cudaGetLastError());
            return;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(grid));
        cfg.blockDim = dim3(static_cast<unsigned>(threads_for(mode)));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        FLW_CUDA(cudaLaunchKernelEx(&cfg, kern, a, carve));
    };
    const bool na8 = a.net.rout[a.net.L - 1] <= 8;
    if (a.act == 0) {
        if (mode == 0) na8 ? go(k_learn<0, 0, 8>) : go(k_learn<0, 0, 16>);
        else if (mode == 1) na8 ? go(k_learn<1, 0, 8>) : go(k_learn<1, 0, 16>);
        else na8 ? go(k_learn<2, 0, 8>) : go(k_learn<2, 0, 16>);
    } else {
        if (mode == 0) na8 ? go(k_learn<0, 1, 8>) : go(k_learn<0, 1, 16>);
        else if (mode == 1) na8 ? go(k_learn<1, 1, 8>) : go(k_learn<1, 1, 16>);
        else na8 ? go(k_learn<2, 1, 8>) : go(k_learn<2, 1, 16>);
    }
}

}  // namespace flw
