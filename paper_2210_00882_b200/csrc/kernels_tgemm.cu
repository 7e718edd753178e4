// Generic warp-specialised tcgen05 GEMM (interface and operand conventions: tgemm.cuh).
//
// One CTA per SM, persistent over work items (128-row tile, BN-column tile, K split):
//   warp 0      TMA producer: one elected lane streams the A / B k-blocks (128-byte rows,
//               SWIZZLE_128B) into an S-stage shared-memory ring (full / empty mbarriers)
//   warp 1      MMA issuer: per k-block BK/UK tcgen05.mma (M=128, N=BN) into one of two TMEM
//               accumulators (double-buffered, so the epilogue of item i overlaps item i+1's
//               MMAs); tcgen05.commit releases the ring slot / hands the accumulator over
//   warps 2-5   epilogue: one accumulator row per thread (TMEM lane quarter = warp % 4),
//               tcgen05.ld in 32-column chunks, fused bias / activation / act' / stores
//
// Shared-memory operand layouts are the canonical UMMA SWIZZLE_128B ones the TMA unit writes
// (cute/atom/mma_traits_sm100.hpp make_umma_desc):
//   K-major : 8-row x 128-byte atoms, atoms along M/N at SBO = 1024 B; the k-th UK-slice of a
//             k-block starts 32 B further (the swizzle is applied on the absolute address bits,
//             so the tiles are 1024-byte aligned)
//   MN-major: 64 bf16 / 32 f32 MN-contiguous elements x 8 K-rows per atom; K-row groups at
//             SBO = 1024 B, MN atoms at LBO = one TMA box (BK rows x 128 B)
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "tgemm.cuh"
#include "umma.cuh"

namespace flw {

namespace {

struct TgArgs {
    int64_t M, N;
    int kblocks, mtiles, ntiles, splits;
    int tma_store;  // bf16 outputs leave through shared memory + TMA stores (map mc)
    // B resident (one N tile, no split-K, B small): the whole B loads once per CTA at shared
    // offset 0 and the ring streams A only
    int bres;
    int nstages;           // ring stages
    uint32_t stage_bytes;  // per stage (A, or A + B)
    uint32_t off_ring;     // first stage
    uint32_t off_stg;      // epilogue output staging
    TgEpilogue epi;
};

constexpr int kTgMaxStages = 8;

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(umma::smem_u32(src))
                 : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(umma::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(umma::smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// SWIZZLE_128B shared-memory descriptor (layout type 2 at bits [61,64), version 1).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// kind::f16 (bf16 / f16) / kind::tf32 instruction descriptor, f32 accumulate, M = 128.
__host__ __device__ constexpr uint32_t idesc_tg(int N, int dt, bool a_mn, bool b_mn) {
    const uint32_t fmt = dt == kTgF32 ? 2u : (dt == kTgF16 ? 0u : 1u);
    return (1u << 4) | (fmt << 7) | (fmt << 10) | (a_mn ? (1u << 15) : 0u) | (b_mn ? (1u << 16) : 0u) |
           (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(128 >> 4) << 24);
}

template <int DT>
__device__ __forceinline__ void mma_tg(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, bool acc) {
    if constexpr (DT == kTgF32) {
        asm volatile(
            "{\n\t.reg .pred p, e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
            "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc ? 1u : 0u));
    } else {
        umma::mma_bf16_warp(tmem_d, adesc, bdesc, idesc, acc);
    }
}

// f32-accurate tanh for the split (rollout) epilogue: an odd minimax polynomial below 0.6,
// 1 - 2 / (exp(2|x|) + 1) above; max relative error ~2e-7 (libdevice tanhf: ~1.2e-7), at a
// third of tanhf's instructions.
__device__ __forceinline__ float tanh_acc(float x) {
    const float ax = fabsf(x);
    if (ax < 0.6f) {
        const float t = x * x;
        float p = -0.00589968f;
        p = fmaf(p, t, 0.020798558f);
        p = fmaf(p, t, -0.053783875f);
        p = fmaf(p, t, 0.13331906f);
        p = fmaf(p, t, -0.33333296f);
        p = fmaf(p, t, 1.0f);
        return x * p;
    }
    const float r = 1.0f - __fdividef(2.0f, __expf(2.0f * ax) + 1.0f);
    return copysignf(r, x);
}

// MUFU tanh (max rel. error ~2^-11, below the bf16 rounding of the stored activation)
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

constexpr int kTgEpiWarps = 8;  // two per TMEM lane quarter, each owning half of the N tile
constexpr int kTgThreads = 32 * (2 + kTgEpiWarps);

template <int BN>
__host__ __device__ constexpr int tg_stages() {
    return BN == 256 ? 4 : (BN == 128 ? 6 : 8);
}
template <int BN>
__host__ __device__ constexpr uint32_t tg_stage_bytes() {
    return 128u * 128u + static_cast<uint32_t>(BN) * 128u;
}

template <int BN, int DT, bool AMN, bool BMN>
__global__ void __launch_bounds__(kTgThreads, 1)
    k_tgemm(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
            const __grid_constant__ CUtensorMap mc, const TgArgs a) {
    const int S = a.nstages;
    const uint32_t kStage = a.stage_bytes;
    constexpr uint32_t kABytes = 128u * 128u;
    constexpr uint32_t kBBlock = static_cast<uint32_t>(BN) * 128u;  // one k-block of B
    constexpr int esz = DT == kTgF32 ? 4 : 2;
    constexpr int BK = 128 / esz;  // K elements per k-block (one 128-byte row)
    constexpr int UK = 32 / esz;   // K elements per MMA
    constexpr int kAtom = 128 / esz;
    constexpr uint32_t kCols = 2 * BN;  // two accumulators
    const uint32_t kStageOff = a.off_stg;  // epilogue output staging: [4 warps][2][32 x 64 B]
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[kTgMaxStages], empty[kTgMaxStages], tfull[2], tempty[2], bfull;
    __shared__ uint32_t tslot;
    __shared__ __align__(16) float sbias[BN];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t items = static_cast<int64_t>(a.mtiles) * a.ntiles * a.splits;

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            umma::mbar_init(&full[i], 1);
            umma::mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            umma::mbar_init(&tfull[i], 1);
            umma::mbar_init(&tempty[i], kTgEpiWarps);
        }
        umma::mbar_init(&bfull, 1);
        umma::fence_barrier_init();
        prefetch_map(&ma);
        prefetch_map(&mb);
    }
    if (w == 1) umma::tmem_alloc<kCols>(&tslot);
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tslot;

    auto decode = [&](int64_t wi, int& mt, int& nt, int& kb0, int& kb1) {
        const int s = static_cast<int>(wi % a.splits);
        const int64_t r = wi / a.splits;
        nt = static_cast<int>(r % a.ntiles);
        mt = static_cast<int>(r / a.ntiles);
        kb0 = static_cast<int>((static_cast<int64_t>(s) * a.kblocks) / a.splits);
        kb1 = static_cast<int>((static_cast<int64_t>(s + 1) * a.kblocks) / a.splits);
        return s;
    };

    if (w == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (umma::elect_one()) {
            int stage = 0;
            uint32_t ph = 0;
            if (a.bres && blockIdx.x < items) {  // the whole B (one N tile), once
                umma::mbar_expect_tx(&bfull, kBBlock * static_cast<uint32_t>(a.kblocks));
                for (int kb = 0; kb < a.kblocks; ++kb) {
                    uint8_t* sb = smem + kb * kBBlock;
                    if constexpr (!BMN) {
                        tma_load_2d(sb, &mb, kb * BK, 0, &bfull);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / kAtom; ++j) tma_load_2d(sb + j * (BK * 128), &mb, j * kAtom, kb * BK, &bfull);
                    }
                }
            }
            for (int64_t wi = blockIdx.x; wi < items; wi += gridDim.x) {
                int mt, nt, kb0, kb1;
                decode(wi, mt, nt, kb0, kb1);
                for (int kb = kb0; kb < kb1; ++kb) {
                    umma::mbar_wait(&empty[stage], ph ^ 1);
                    uint8_t* sa = smem + a.off_ring + stage * kStage;
                    uint8_t* sb = sa + kABytes;
                    umma::mbar_expect_tx(&full[stage], kStage);
                    if constexpr (!AMN) {
                        tma_load_2d(sa, &ma, kb * BK, mt * 128, &full[stage]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 128 / kAtom; ++j)
                            tma_load_2d(sa + j * (BK * 128), &ma, mt * 128 + j * kAtom, kb * BK, &full[stage]);
                    }
                    if (a.bres) {
                    } else if constexpr (!BMN) {
                        tma_load_2d(sb, &mb, kb * BK, nt * BN, &full[stage]);
                    } else {
#pragma unroll
                        for (int j = 0; j < BN / kAtom; ++j)
                            tma_load_2d(sb + j * (BK * 128), &mb, nt * BN + j * kAtom, kb * BK, &full[stage]);
                    }
                    if (++stage == S) {
                        stage = 0;
                        ph ^= 1;
                    }
                }
            }
        }
    } else if (w == 1) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = idesc_tg(BN, DT, AMN, BMN);
        int stage = 0;
        uint32_t ph = 0, tph[2] = {0, 0};
        int acc = 0;
        const uint32_t sbase = umma::smem_u32(smem);
        if (a.bres && blockIdx.x < items) umma::mbar_wait(&bfull, 0);
        for (int64_t wi = blockIdx.x; wi < items; wi += gridDim.x) {
            int mt, nt, kb0, kb1;
            decode(wi, mt, nt, kb0, kb1);
            umma::mbar_wait(&tempty[acc], tph[acc] ^ 1);
            tph[acc] ^= 1;
            umma::fence_after_sync();
            const uint32_t dt = tmem + static_cast<uint32_t>(acc * BN);
            for (int kb = kb0; kb < kb1; ++kb) {
                umma::mbar_wait(&full[stage], ph);
                umma::fence_after_sync();
                const uint32_t sa = sbase + a.off_ring + stage * kStage;
                const uint32_t sb = a.bres ? sbase + kb * kBBlock : sa + kABytes;
#pragma unroll
                for (int k = 0; k < BK / UK; ++k) {
                    const uint64_t ad = AMN ? desc_sw128(sa + k * (UK * 128), BK * 128, 1024)
                                            : desc_sw128(sa + k * 32, 16, 1024);
                    const uint64_t bd = BMN ? desc_sw128(sb + k * (UK * 128), BK * 128, 1024)
                                            : desc_sw128(sb + k * 32, 16, 1024);
                    mma_tg<DT>(dt, ad, bd, idesc, kb > kb0 || k > 0);
                }
                umma::commit_warp(&empty[stage]);  // the slot is free once these MMAs read it
                if (++stage == S) {
                    stage = 0;
                    ph ^= 1;
                }
            }
            umma::commit_warp(&tfull[acc]);
            acc ^= 1;
        }
    } else {
        // ------------------------------------------------------------------ epilogue
        const int q = w & 3;              // TMEM lane quarter
        const int hn = (w - 2) >> 2;      // which half of the N tile
        const int et = threadIdx.x - 64;  // 0..255 over the eight epilogue warps
        const TgEpilogue& e = a.epi;
        const int64_t m_store = e.m_store >= 0 ? e.m_store : a.M;
        const int64_t n_store = e.n_store >= 0 ? e.n_store : a.N;
        const bool use_bias = e.mode == kTgBias || e.mode == kTgBiasAct || e.mode == kTgSplit3;
        uint32_t tph[2] = {0, 0};
        int acc = 0;
        for (int64_t wi = blockIdx.x; wi < items; wi += gridDim.x) {
            int mt, nt, kb0, kb1;
            const int s = decode(wi, mt, nt, kb0, kb1);
            const int64_t n0 = static_cast<int64_t>(nt) * BN;
            if (use_bias) {  // this item's bias slice, staged once (named barrier: epilogue warps)
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
                for (int i = et; i < BN; i += 256) sbias[i] = n0 + i < n_store ? e.bias[n0 + i] : 0.0f;
                asm volatile("bar.sync 1, 256;\n" ::: "memory");
            }
            umma::mbar_wait(&tfull[acc], tph[acc]);
            tph[acc] ^= 1;
            umma::fence_after_sync();
            const int64_t m = static_cast<int64_t>(mt) * 128 + 32 * q + lane;
            const uint32_t dt = tmem + (static_cast<uint32_t>(32 * q) << 16) + static_cast<uint32_t>(acc * BN);
            const bool mok = m < m_store;
#pragma unroll 1
            for (int c0 = hn * (BN / 2); c0 < (hn + 1) * (BN / 2); c0 += 32) {
                if (n0 + c0 >= n_store) break;  // warp-uniform
                float v[32];
                umma::tmem_ld16(dt + c0, v);
                umma::tmem_ld16(dt + c0 + 16, v + 16);
                const int64_t nb = n0 + c0;
                const int nv = n_store - nb < 32 ? static_cast<int>(n_store - nb) : 32;
                uint4 hv[4];  // act' input row slice, loaded while the TMEM load is in flight
                if (e.mode == kTgActGrad && mok) {
                    const __nv_bfloat16* hr = e.h + m * e.ldh + nb;
                    if (nv == 32 && (e.ldh & 7) == 0) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) hv[j] = __ldg(reinterpret_cast<const uint4*>(hr + 8 * j));
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint32_t w4[4];
#pragma unroll
                            for (int i = 0; i < 4; ++i) {
                                const int c = 8 * j + 2 * i;
                                const float x0 = c < nv ? __bfloat162float(hr[c]) : 0.0f;
                                const float x1 = c + 1 < nv ? __bfloat162float(hr[c + 1]) : 0.0f;
                                w4[i] = umma::pack_bf16x2(x0, x1);
                            }
                            hv[j] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
                        }
                    }
                }
                umma::tmem_ld_wait();
                // (TMA-stored chunks keep every lane: the store clips rows beyond m_store)
                if (!mok && !(a.tma_store && (e.mode == kTgBiasAct || e.mode == kTgActGrad))) continue;
                if (use_bias) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 b4 = *reinterpret_cast<const float4*>(sbias + c0 + j);
                        v[j] += b4.x;
                        v[j + 1] += b4.y;
                        v[j + 2] += b4.z;
                        v[j + 3] += b4.w;
                    }
                }
                if (e.mode == kTgStoreF32 || e.mode == kTgBias) {
                    float* dst = e.c32 + static_cast<int64_t>(s) * e.split_stride + m * e.ldc32 + nb;
                    if (nv == 32 && (e.ldc32 & 3) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4)
                            *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                    } else {  // (static indices keep v[] in registers)
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (j < nv) dst[j] = v[j];
                    }
                    continue;
                }
                if (e.mode == kTgSplit3) {  // f32-accurate activation, split into f16 hi + lo
                    uint32_t hi[16], lo[16];
#pragma unroll
                    for (int j = 0; j < 32; j += 2) {
                        const float y0 = e.act == 0 ? tanh_acc(v[j]) : fmaxf(v[j], 0.0f);
                        const float y1 = e.act == 0 ? tanh_acc(v[j + 1]) : fmaxf(v[j + 1], 0.0f);
                        const __half h0 = __float2half_rn(y0), h1 = __float2half_rn(y1);
                        const __half l0 = __float2half_rn(y0 - __half2float(h0));
                        const __half l1 = __float2half_rn(y1 - __half2float(h1));
                        hi[j / 2] = static_cast<uint32_t>(__half_as_ushort(h0)) |
                                    (static_cast<uint32_t>(__half_as_ushort(h1)) << 16);
                        lo[j / 2] = static_cast<uint32_t>(__half_as_ushort(l0)) |
                                    (static_cast<uint32_t>(__half_as_ushort(l1)) << 16);
                    }
                    __half* d = e.c16h + m * e.ldc16 + nb;
                    if (nv == 32 && (e.ldc16 & 7) == 0 && (e.seg & 7) == 0) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint4 h4 = make_uint4(hi[4 * j], hi[4 * j + 1], hi[4 * j + 2], hi[4 * j + 3]);
                            *reinterpret_cast<uint4*>(d + 8 * j) = h4;
                            *reinterpret_cast<uint4*>(d + e.seg + 8 * j) =
                                make_uint4(lo[4 * j], lo[4 * j + 1], lo[4 * j + 2], lo[4 * j + 3]);
                            *reinterpret_cast<uint4*>(d + 2 * e.seg + 8 * j) = h4;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            if (j < nv) {
                                const unsigned short hs = static_cast<unsigned short>(hi[j / 2] >> (16 * (j & 1)));
                                const unsigned short ls = static_cast<unsigned short>(lo[j / 2] >> (16 * (j & 1)));
                                d[j] = __ushort_as_half(hs);
                                d[e.seg + j] = __ushort_as_half(ls);
                                d[2 * e.seg + j] = __ushort_as_half(hs);
                            }
                        }
                    }
                    continue;
                }
                if (e.mode == kTgBiasAct) {
                    if (e.act == 0) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = tanh_approx(v[j]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) v[j] = fmaxf(v[j], 0.0f);
                    }
                    if (e.c32) {
                        float* d32 = e.c32 + m * e.ldc32 + nb;
                        if (nv == 32 && (e.ldc32 & 3) == 0) {
#pragma unroll
                            for (int j = 0; j < 32; j += 4)
                                *reinterpret_cast<float4*>(d32 + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (j < nv) d32[j] = v[j];
                        }
                    }
                    if (!e.c16) continue;  // f32 output only
                } else {  // kTgActGrad: acc * act'(h), h = the activation output (bf16)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&hv[j]);
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float2 y = __bfloat1622float2(h2[i]);
                            const int c = 8 * j + 2 * i;
                            if (e.act == 0) {
                                v[c] *= 1.0f - y.x * y.x;
                                v[c + 1] *= 1.0f - y.y * y.y;
                            } else {
                                v[c] = y.x > 0.0f ? v[c] : 0.0f;
                                v[c + 1] = y.y > 0.0f ? v[c + 1] : 0.0f;
                            }
                        }
                    }
                }
                if (a.tma_store) {
                    // this warp's 32 rows x 32 columns (64 B per row) into its staging buffer in
                    // the SWIZZLE_64B layout (16-byte chunk k of row r at k ^ ((r >> 1) & 3)),
                    // then one TMA store; the other buffer's store may still be reading
                    uint8_t* stg = smem + kStageOff + ((w - 2) * 2 + (c0 >> 5 & 1)) * 2048;
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        *reinterpret_cast<uint4*>(stg + lane * 64 + ((k ^ ((lane >> 1) & 3)) << 4)) =
                            make_uint4(umma::pack_bf16x2(v[8 * k], v[8 * k + 1]),
                                       umma::pack_bf16x2(v[8 * k + 2], v[8 * k + 3]),
                                       umma::pack_bf16x2(v[8 * k + 4], v[8 * k + 5]),
                                       umma::pack_bf16x2(v[8 * k + 6], v[8 * k + 7]));
                    umma::fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&mc, static_cast<int>(nb), static_cast<int>(mt * 128 + 32 * q), stg);
                        umma::bulk_commit();
                    }
                    continue;
                }
                __nv_bfloat16* d16 = e.c16 + m * e.ldc16 + nb;
                if (nv == 32 && (e.ldc16 & 7) == 0) {
#pragma unroll
                    for (int j = 0; j < 32; j += 8)
                        *reinterpret_cast<uint4*>(d16 + j) =
                            make_uint4(umma::pack_bf16x2(v[j], v[j + 1]), umma::pack_bf16x2(v[j + 2], v[j + 3]),
                                       umma::pack_bf16x2(v[j + 4], v[j + 5]), umma::pack_bf16x2(v[j + 6], v[j + 7]));
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (j < nv) d16[j] = __float2bfloat16(v[j]);
                }
            }
            umma::fence_before_sync();
            __syncwarp();
            if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(umma::smem_u32(&tempty[acc])) : "memory");
            acc ^= 1;
        }
        if (a.tma_store && lane == 0) umma::bulk_wait_all();  // the staged outputs are written
        __syncwarp();
    }
    umma::fence_before_sync();
    __syncthreads();
    if (w == 1) umma::tmem_free<kCols>(tmem);
}

// ---------------------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        FLW_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(Errc::Runtime, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

CUtensorMap make_map(const TgOperand& o, uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    const int esz = o.dt == kTgF32 ? 4 : 2;
    if ((reinterpret_cast<uintptr_t>(o.ptr) & 15) != 0 || (o.ld * esz) % 16 != 0)
        throw Error(Errc::Config, "tgemm: operand base / row stride must be 16-byte aligned");
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(o.cols), static_cast<cuuint64_t>(o.rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(o.ld * esz)};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    const CUtensorMapDataType ty = o.dt == kTgF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : (o.dt == kTgF16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
    const CUresult r = encode_fn()(&m, ty, 2,
                                   const_cast<void*>(o.ptr), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(Errc::Runtime, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    return m;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        FLW_CUDA(cudaGetDevice(&dev));
        FLW_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

template <int BN, int DT, bool AMN, bool BMN>
void launch_tg(cudaStream_t s, const TgOperand& A, const TgOperand& B, TgArgs a, int grid_cap) {
    constexpr int esz = DT == kTgF32 ? 4 : 2;
    constexpr uint32_t BK = 128 / esz, atom = 128 / esz;
    const CUtensorMap ma = AMN ? make_map(A, atom, BK) : make_map(A, BK, 128);
    const CUtensorMap mb = BMN ? make_map(B, atom, BK) : make_map(B, BK, BN);
    // A/B option (FLW_TG_TMA_STORE=1): bf16 outputs leave through shared memory and TMA stores
    // (32 x 32 boxes, SWIZZLE_64B). Measured: H = 256 layer-wise learn slower (forward GEMM 42 ->
    // 50 us), MAPPO n = 64 2% faster - off by default.
    static const bool tma_store_on = std::getenv("FLW_TG_TMA_STORE") != nullptr;
    const TgEpilogue& e = a.epi;
    CUtensorMap mc = ma;
    a.tma_store = 0;
    if (tma_store_on && (e.mode == kTgBiasAct || e.mode == kTgActGrad) && !e.c32 && e.c16 &&
        (reinterpret_cast<uintptr_t>(e.c16) & 15) == 0 && (e.ldc16 * 2) % 16 == 0) {
        const int64_t ms = e.m_store >= 0 ? e.m_store : a.M, ns = e.n_store >= 0 ? e.n_store : a.N;
        mc = make_map(TgOperand{e.c16, ms, ns, e.ldc16, kTgBF16}, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        a.tma_store = 1;
    }
    constexpr uint32_t kBBlock = static_cast<uint32_t>(BN) * 128u, kAB = 128u * 128u;
    constexpr uint32_t kBudget = 227u * 1024u - 4096u;  // dynamic shared memory (static: barriers, bias)
    const uint32_t bbytes = kBBlock * static_cast<uint32_t>(a.kblocks);
    a.bres = a.ntiles == 1 && a.splits == 1 && a.mtiles > sm_count() && bbytes <= 128u * 1024u;
    if (a.bres) {
        a.off_ring = (bbytes + 1023u) / 1024u * 1024u;
        a.stage_bytes = kAB;
        a.nstages = static_cast<int>(
            std::min<uint32_t>(kTgMaxStages, (kBudget - a.off_ring - (a.tma_store ? 32768u : 0u) - 1024u) / kAB));
    } else {
        a.off_ring = 0;
        a.stage_bytes = tg_stage_bytes<BN>();
        a.nstages = tg_stages<BN>();
    }
    a.off_stg = a.off_ring + static_cast<uint32_t>(a.nstages) * a.stage_bytes;
    const uint32_t stg = a.tma_store ? 2048u * 2 * kTgEpiWarps : 0u;  // [warp][2][32 x 64 B]
    const size_t smem = static_cast<size_t>(a.off_stg) + stg + 1024;
    auto kern = k_tgemm<BN, DT, AMN, BMN>;
    FLW_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    const int64_t items = static_cast<int64_t>(a.mtiles) * a.ntiles * a.splits;
    const int cap = grid_cap > 0 ? grid_cap : sm_count();
    const int grid = static_cast<int>(std::min<int64_t>(items, cap));
    kern<<<grid, kTgThreads, smem, s>>>(ma, mb, mc, a);
    FLW_CUDA(cudaGetLastError());
}

template <int BN, int DT>
void dispatch_major(cudaStream_t s, const TgOperand& A, bool a_mn, const TgOperand& B, bool b_mn, const TgArgs& a,
                    int cap) {
    if (!a_mn && !b_mn) launch_tg<BN, DT, false, false>(s, A, B, a, cap);
    else if (!a_mn && b_mn) launch_tg<BN, DT, false, true>(s, A, B, a, cap);
    else if (a_mn && !b_mn) launch_tg<BN, DT, true, false>(s, A, B, a, cap);
    else launch_tg<BN, DT, true, true>(s, A, B, a, cap);
}

}  // namespace

void tgemm(cudaStream_t s, const TgOperand& A, bool a_mn, const TgOperand& B, bool b_mn, int64_t M, int64_t N,
           int64_t K, int splits, const TgEpilogue& epi, int bn, int grid_cap) {
    if (A.dt != B.dt) throw Error(Errc::Config, "tgemm: A and B must share the element type");
    // 32-bit MN-major operands need the SWIZZLE_128B_BASE32B canonical layout, not this one
    if (A.dt == kTgF32 && (a_mn || b_mn)) throw Error(Errc::Config, "tgemm: tf32 operands must both be K-major");
    if (bn != 64 && bn != 128 && bn != 256) throw Error(Errc::Config, "tgemm: bn must be 64, 128 or 256");
    if (M <= 0 || N <= 0 || K <= 0) return;
    const int BK = A.dt == kTgF32 ? 32 : 64;
    TgArgs a{};
    a.M = M;
    a.N = N;
    a.kblocks = static_cast<int>((K + BK - 1) / BK);
    a.mtiles = static_cast<int>((M + 127) / 128);
    a.ntiles = static_cast<int>((N + bn - 1) / bn);
    a.splits = std::max(1, std::min(splits, a.kblocks));
    if (a.splits > 1 && epi.mode != kTgStoreF32) throw Error(Errc::Config, "tgemm: split-K needs the f32 partial epilogue");
    a.epi = epi;
    auto go = [&](auto bnc) {
        constexpr int BNc = decltype(bnc)::value;
        if (A.dt == kTgF32) dispatch_major<BNc, kTgF32>(s, A, a_mn, B, b_mn, a, grid_cap);
        else if (A.dt == kTgF16) dispatch_major<BNc, kTgF16>(s, A, a_mn, B, b_mn, a, grid_cap);
        else dispatch_major<BNc, kTgBF16>(s, A, a_mn, B, b_mn, a, grid_cap);
    };
    if (bn == 64) go(std::integral_constant<int, 64>{});
    else if (bn == 128) go(std::integral_constant<int, 128>{});
    else go(std::integral_constant<int, 256>{});
}

}  // namespace flw

// ---------------------------------------------------------------------------- self-test (C-ABI)
// D = op(A) op(B) through tgemm with the f32 partial epilogue; the K splits are summed here.
// a_mn: A given as [K, M] (else [M, K]); b_mn: B given as [K, N] (else [N, K]). tf32: 1 operands
// stay f32 (kind::tf32), 2 rounded to f16, 0 rounded to bf16 (kind::f16).
extern "C" int flw_selftest_tgemm(int64_t M, int64_t N, int64_t K, int a_mn, int b_mn, int tf32, int splits, int bn,
                                  const float* A, const float* B, float* D) {
    using namespace flw;
    try {
        const int64_t ar = a_mn ? K : M, ac = a_mn ? M : K, br = b_mn ? K : N, bc = b_mn ? N : K;
        const int dt = tf32 == 1 ? kTgF32 : (tf32 == 2 ? kTgF16 : kTgBF16);
        const int esz = dt == kTgF32 ? 4 : 2;
        const int64_t ald = (ac * esz + 15) / 16 * 16 / esz, bld = (bc * esz + 15) / 16 * 16 / esz;
        std::vector<uint8_t> ha(static_cast<size_t>(ar * ald * esz), 0), hb(static_cast<size_t>(br * bld * esz), 0);
        for (int64_t r = 0; r < ar; ++r)
            for (int64_t c = 0; c < ac; ++c) {
                if (dt == kTgF32) reinterpret_cast<float*>(ha.data())[r * ald + c] = A[r * ac + c];
                else if (dt == kTgF16) reinterpret_cast<__half*>(ha.data())[r * ald + c] = __float2half_rn(A[r * ac + c]);
                else reinterpret_cast<__nv_bfloat16*>(ha.data())[r * ald + c] = __float2bfloat16(A[r * ac + c]);
            }
        for (int64_t r = 0; r < br; ++r)
            for (int64_t c = 0; c < bc; ++c) {
                if (dt == kTgF32) reinterpret_cast<float*>(hb.data())[r * bld + c] = B[r * bc + c];
                else if (dt == kTgF16) reinterpret_cast<__half*>(hb.data())[r * bld + c] = __float2half_rn(B[r * bc + c]);
                else reinterpret_cast<__nv_bfloat16*>(hb.data())[r * bld + c] = __float2bfloat16(B[r * bc + c]);
            }
        void *da = nullptr, *db = nullptr;
        float* dd = nullptr;
        const int BK = dt == kTgF32 ? 32 : 64;
        const int sp = std::max(1, std::min<int>(splits, static_cast<int>((K + BK - 1) / BK)));
        FLW_CUDA(cudaMalloc(&da, ha.size()));
        FLW_CUDA(cudaMalloc(&db, hb.size()));
        FLW_CUDA(cudaMalloc(&dd, static_cast<size_t>(sp * M * N) * sizeof(float)));
        FLW_CUDA(cudaMemcpy(da, ha.data(), ha.size(), cudaMemcpyHostToDevice));
        FLW_CUDA(cudaMemcpy(db, hb.data(), hb.size(), cudaMemcpyHostToDevice));
        FLW_CUDA(cudaMemset(dd, 0, static_cast<size_t>(sp * M * N) * sizeof(float)));
        TgEpilogue e;
        e.mode = kTgStoreF32;
        e.c32 = dd;
        e.ldc32 = N;
        e.split_stride = M * N;
        tgemm(nullptr, TgOperand{da, ar, ac, ald, dt}, a_mn != 0, TgOperand{db, br, bc, bld, dt}, b_mn != 0,
              M, N, K, sp, e, bn);
        std::vector<float> part(static_cast<size_t>(sp * M * N));
        FLW_CUDA(cudaDeviceSynchronize());
        FLW_CUDA(cudaMemcpy(part.data(), dd, part.size() * sizeof(float), cudaMemcpyDeviceToHost));
        for (int64_t i = 0; i < M * N; ++i) {
            float t = 0.0f;
            for (int s2 = 0; s2 < sp; ++s2) t += part[static_cast<size_t>(s2 * M * N + i)];
            D[i] = t;
        }
        cudaFree(da);
        cudaFree(db);
        cudaFree(dd);
        return 0;
    } catch (const std::exception& ex) {
        fprintf(stderr, "flw_selftest_tgemm: %s\n", ex.what());
        return 3;
    }
}

// Diagnostic: mean ms per tgemm launch for one shape / epilogue (synthetic operands, CUDA events
// after warm-up). mode: kTgStoreF32, kTgBiasAct (bf16 out), kTgSplit3 (f16 hi|lo|hi out).
extern "C" int flw_bench_tgemm(int64_t M, int64_t N, int64_t K, int dt, int mode, int bn, int iters, double* ms) {
    using namespace flw;
    try {
        const int esz = dt == kTgF32 ? 4 : 2;
        const int64_t lda = (K * esz + 15) / 16 * 16 / esz, ldb = (N * esz + 15) / 16 * 16 / esz;
        void *da = nullptr, *db = nullptr, *dc = nullptr;
        float* bias = nullptr;
        FLW_CUDA(cudaMalloc(&da, static_cast<size_t>(M * lda * esz)));
        FLW_CUDA(cudaMalloc(&db, static_cast<size_t>(K * ldb * esz)));
        FLW_CUDA(cudaMalloc(&dc, static_cast<size_t>(M * 3 * ((N + 63) / 64 * 64)) * 4));
        FLW_CUDA(cudaMalloc(&bias, static_cast<size_t>(N) * 4));
        FLW_CUDA(cudaMemset(da, 0, static_cast<size_t>(M * lda * esz)));
        FLW_CUDA(cudaMemset(db, 0, static_cast<size_t>(K * ldb * esz)));
        FLW_CUDA(cudaMemset(bias, 0, static_cast<size_t>(N) * 4));
        TgEpilogue e;
        e.mode = mode;
        e.bias = bias;
        if (mode == kTgStoreF32) {
            e.c32 = static_cast<float*>(dc);
            e.ldc32 = N;
        } else if (mode == kTgSplit3) {
            e.c16h = static_cast<__half*>(dc);
            e.seg = (N + 63) / 64 * 64;
            e.ldc16 = 3 * e.seg;
        } else {
            e.c16 = static_cast<__nv_bfloat16*>(dc);
            e.ldc16 = (N + 7) / 8 * 8;
        }
        auto run = [&] {
            tgemm(nullptr, TgOperand{da, M, K, lda, dt}, false, TgOperand{db, K, N, ldb, dt}, dt != kTgF32, M, N, K, 1, e,
                  bn);
        };
        for (int i = 0; i < 3; ++i) run();
        cudaEvent_t a, b;
        FLW_CUDA(cudaEventCreate(&a));
        FLW_CUDA(cudaEventCreate(&b));
        FLW_CUDA(cudaEventRecord(a, nullptr));
        for (int i = 0; i < iters; ++i) run();
        FLW_CUDA(cudaEventRecord(b, nullptr));
        FLW_CUDA(cudaEventSynchronize(b));
        float t = 0.0f;
        FLW_CUDA(cudaEventElapsedTime(&t, a, b));
        *ms = t / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(da);
        cudaFree(db);
        cudaFree(dc);
        cudaFree(bias);
        return 0;
    } catch (const std::exception& ex) {
        fprintf(stderr, "flw_bench_tgemm: %s\n", ex.what());
        return 3;
    }
}
