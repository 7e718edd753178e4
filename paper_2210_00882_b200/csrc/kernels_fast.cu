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

#include "common.cuh"
#include "fast.cuh"
#include "umma.cuh"

namespace flw {

namespace {

constexpr int kRows = 128;
constexpr int kMaxW = 64;
constexpr int kThreads = 256;
constexpr int kDbSlices = 4;  // db column sums: 4 threads per column, 32 rows each

struct Smem {  // carve-up of dynamic shared memory (byte offsets)
    uint32_t wt[kMaxLayers], x, h[kMaxLayers], dz[2], bias, dbacc, loss, total;
};

__host__ __device__ inline uint32_t align_up(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline Smem carve(const FastNet& n) {
    Smem s{};
    uint32_t off = 0;
    for (int l = 0; l < n.L; ++l) {
        s.wt[l] = off;
        off = align_up(off + static_cast<uint32_t>(n.dout[l] * n.din[l] * 2), 128);
    }
    s.x = off;
    off = align_up(off + kRows * n.din[0] * 2, 128);
    for (int l = 0; l + 1 < n.L; ++l) {
        s.h[l] = off;
        off = align_up(off + static_cast<uint32_t>(kRows * n.dout[l] * 2), 128);
    }
    for (int i = 0; i < 2; ++i) {
        s.dz[i] = off;
        off = align_up(off + kRows * kMaxW * 2, 128);
    }
    s.bias = off;
    off += kMaxLayers * kMaxW * 4;
    s.dbacc = off;
    off += kDbSlices * kMaxLayers * kMaxW * 4;  // one slice per row quarter
    s.loss = off;
    off += 8 * 3 * 4;
    // slack: M=64 MN-major reads of narrow tiles run past their end (rows >= din are ignored)
    s.total = off + 2048;
    return s;
}

// MUFU tanh (max rel. error ~2^-11): the activation is rounded to bf16 (2^-8) right after.
__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float act_fwd(float z, int act) { return act == 0 ? tanh_fast(z) : (z > 0.0f ? z : 0.0f); }

__global__ void __launch_bounds__(kThreads, 1) k_fast_mlp(FastLearnArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar, hbar;
    __shared__ uint32_t tslot;
    uint32_t hphase = 0;
    const FastNet& n = a.net;
    const Smem S = carve(n);
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    const int quad = w & 3, half = w >> 2;
    const int r = 32 * quad + lane;  // tile row == TMEM lane
    const int L = n.L;
    float* bias = reinterpret_cast<float*>(smem + S.bias);
    float* dbacc = reinterpret_cast<float*>(smem + S.dbacc);

    // ---- weights (once per CTA): W_l^T as [dout x din] K-major B tiles, zero padded; copied
    // with 16-byte loads from the pre-built image (k_build_wimg) that every CTA shares via L2
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.wimg);
        uint4* dst = reinterpret_cast<uint4*>(smem);
        for (uint32_t i = t; i < S.x / 16; i += kThreads) dst[i] = src[i];
    }
    for (int l = 0; l < L; ++l) {
        const int ro = n.rout[l];
        for (int o = t; o < kMaxW; o += kThreads) bias[l * kMaxW + o] = o < ro ? a.params[n.boff[l] + o] : 0.0f;
    }
    for (int i = t; i < kDbSlices * kMaxLayers * kMaxW; i += kThreads) dbacc[i] = 0.0f;
    umma::fence_async_smem();
    if (w == 0) umma::tmem_alloc<512>(&tslot);
    if (t == 0) {
        umma::mbar_init(&bar, 1);
        umma::mbar_init(&hbar, 1);
        umma::fence_barrier_init();
    }
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t tmem = tslot;
    const uint32_t lane_base = static_cast<uint32_t>(32 * quad) << 16;
    const uint32_t sbase = umma::smem_u32(smem);
    uint32_t phase = 0;
    float pl_acc = 0.0f, vl_acc = 0.0f, en_acc = 0.0f;
    bool first = true;
    const int64_t ntiles = (a.rows + kRows - 1) / kRows;

    // Input rows are fetched one tile ahead into registers (this thread's 8-column chunks of
    // its row), so the HBM latency of tile i+1 hides behind tile i's 2L GEMM stages.
    constexpr int kXRegs = kMaxW / 2;
    float xnext[kXRegs];
    auto fetch_x = [&](int64_t tl) {
        const int64_t rw = tl * kRows + r;
        const bool ok = tl < ntiles && rw < a.rows;
#pragma unroll
        for (int k = 0; k < kXRegs / 8; ++k) {
            const int c0 = 8 * half + 16 * k;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = c0 + j;
                xnext[8 * k + j] = (ok && c < a.in_cols) ? a.X[rw * a.in_cols + c] : 0.0f;
            }
        }
    };
    fetch_x(blockIdx.x);

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row = tile * kRows + r;
        const bool valid = row < a.rows;
        // ---- input tile (f32 -> bf16), zero padded columns and rows; halves split 8-col chunks
#pragma unroll
        for (int k = 0; k < kXRegs / 8; ++k) {
            const int c0 = 8 * half + 16 * k;
            float v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = xnext[8 * k + j];
            if (c0 < n.din[0]) umma::st_row8(smem + S.x, n.din[0], r, c0, v);
        }
        fetch_x(tile + gridDim.x);
        // per-row learn inputs, issued now and consumed by the loss epilogue after the forward
        int act_r = 0;
        float lpo_r = 0.0f, adv_r = 0.0f, ret_r = 0.0f, val_r = 0.0f;
        if (a.mode == 1 && half == 0 && valid) {
            ret_r = a.kind == kNetPolicyPpo ? 0.0f : a.ret[row];
            if (a.kind != kNetCritic) act_r = a.actions[row];
            if (a.kind == kNetPolicyPpo) {
                lpo_r = a.logp_old[row];
                adv_r = a.adv[row];
            }
            if (a.kind == kNetPolicyA3c) val_r = a.values_in[row];
        }
        // hidden-activation region [S.h[0], S.h[L-2] + size): contiguous in shared memory
        const uint32_t hbytes = L > 1 ? S.dz[0] - S.h[0] : 0u;
        const bool reuse = a.hload && a.mode == 1 && hbytes > 0;
        if (t == 0 && hbytes > 0) {
            if (a.mode == 0) umma::bulk_wait_read();  // previous tile's save has read the region
            if (reuse) {  // saved tile -> shared memory via the TMA engine (arrives on hbar)
                umma::mbar_expect_tx(&hbar, hbytes);
                const uint8_t* src = a.hsave + static_cast<size_t>(tile) * hbytes;
                for (uint32_t o = 0; o < hbytes; o += 16384u)
                    umma::bulk_g2s(smem + S.h[0] + o, src + o, min(16384u, hbytes - o), &hbar);
            }
        }
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        // ---- forward (skipped when the critic's activations are reused from the values pass)
        float out[16];
        if (reuse) {
            umma::mbar_wait(&hbar, hphase);
            hphase ^= 1;
            out[0] = valid ? a.values_in[row] : 0.0f;
        }
        for (int l = 0; l < (reuse ? 0 : L); ++l) {
            const int di = n.din[l], dout = n.dout[l];
            const uint32_t in_tile = l == 0 ? sbase + S.x : sbase + S.h[l - 1];
            if (t == 0) {
                umma::fence_after_sync();
                const uint32_t idesc = umma::idesc_bf16(128, dout, false, false);
                for (int kb = 0; kb < di / 16; ++kb)
                    umma::mma_bf16(tmem, umma::desc_kmajor(in_tile, di, kb),
                                   umma::desc_kmajor(sbase + S.wt[l], di, kb), idesc, kb > 0);
                umma::commit(&bar);
            }
            umma::mbar_wait(&bar, phase);
            phase ^= 1;
            umma::fence_after_sync();
            const bool last = l + 1 == L;
            for (int c0 = 16 * half; c0 < dout; c0 += 32) {
                float z[16];
                umma::tmem_ld16(tmem + lane_base + c0, z);
                umma::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 16; ++j) z[j] += bias[l * kMaxW + c0 + j];
                if (!last) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) z[j] = act_fwd(z[j], a.act);
                    umma::st_row8(smem + S.h[l], dout, r, c0, z);
                    umma::st_row8(smem + S.h[l], dout, r, c0 + 8, z + 8);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) out[j] = z[j];
                }
            }
            umma::fence_async_smem();
            umma::fence_before_sync();
            __syncthreads();
        }
        // values pass: hand this tile's hidden activations to the learn kernel (async bulk store)
        if (a.mode == 0 && a.hsave && t == 0 && hbytes > 0 && tile < a.save_tiles) {
            uint8_t* dst = a.hsave + static_cast<size_t>(tile) * hbytes;
            for (uint32_t o = 0; o < hbytes; o += 16384u)
                umma::bulk_s2g(dst + o, smem + S.h[0] + o, min(16384u, hbytes - o));
            umma::bulk_commit();
        }
        // ---- loss epilogue (rl.cpp:137-202 semantics, f32) -> dZ_{L-1}; the output layer is one
        // 16-column chunk, owned by the half-0 warps.
        if (half == 0) {
            float dz[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) dz[j] = 0.0f;
            if (a.mode == 0) {
                if (valid) {
                    if (a.split_rows >= 0 && row >= a.split_rows)
                        a.values_out2[row - a.split_rows] = out[0];
                    else
                        a.values_out[row] = out[0];
                }
            } else if (valid) {
                if (a.kind == kNetCritic) {  // value MSE: dV = 2 c_v (V - R) / N
                    float verr = out[0] - ret_r;
                    dz[0] = static_cast<float>(2.0 * a.value_coef * a.inv_n) * verr;
                    vl_acc += static_cast<float>(a.value_coef * a.inv_n) * verr * verr;
                } else {  // policy: clipped surrogate (PPO) or A3C policy gradient, + entropy bonus
                    const int A = n.rout[L - 1];
                    float mx = out[0];
                    for (int j = 1; j < A; ++j) mx = fmaxf(mx, out[j]);
                    float den = 0.0f;
                    for (int j = 0; j < A; ++j) den += expf(out[j] - mx);
                    const float lden = logf(den);
                    float p[16], lp[16], H = 0.0f;
                    for (int j = 0; j < A; ++j) {
                        lp[j] = out[j] - mx - lden;
                        p[j] = expf(lp[j]);
                        H -= p[j] * lp[j];
                    }
                    const int act = act_r;
                    const float inv_n = static_cast<float>(a.inv_n);
                    float coef;
                    if (a.kind == kNetPolicyPpo) {
                        float adv = adv_r;
                        if (a.adv_stats) {
                            const double sd = a.adv_stats[1];
                            if (!(sd < 1e-8)) adv = static_cast<float>((adv - a.adv_stats[0]) / (sd + 1e-8));
                        }
                        const float ratio = expf(lp[act] - lpo_r);
                        const float clipped = fminf(fmaxf(ratio, 1.0f - a.clip_eps), 1.0f + a.clip_eps);
                        const float s1 = ratio * adv, s2 = clipped * adv;
                        pl_acc -= fminf(s1, s2) * inv_n;
                        coef = s1 <= s2 ? -inv_n * ratio * adv : 0.0f;
                    } else {  // A3C: advantage R - V (rl.cpp:188)
                        const float adv = ret_r - val_r;
                        pl_acc -= lp[act] * adv * inv_n;
                        coef = -inv_n * adv;
                    }
                    en_acc += H * inv_n;
                    const float eci = static_cast<float>(a.entropy_coef) * inv_n;
                    for (int j = 0; j < A; ++j)
                        dz[j] = coef * ((j == act ? 1.0f : 0.0f) - p[j]) + eci * p[j] * (lp[j] + H);
                }
            }
            if (a.mode == 1) {
                umma::st_row8(smem + S.dz[0], n.dout[L - 1], r, 0, dz);
                umma::st_row8(smem + S.dz[0], n.dout[L - 1], r, 8, dz + 8);
            }
        }
        if (a.mode == 0) continue;  // forward only: the next tile reuses the same buffers safely
        int cur = 0;
        umma::fence_async_smem();
        umma::fence_before_sync();
        __syncthreads();
        // ---- backward
        for (int l = L - 1; l >= 0; --l) {
            const int di = n.din[l], dout = n.dout[l];
            const uint32_t hin = l == 0 ? sbase + S.x : sbase + S.h[l - 1];
            const uint32_t dzt = sbase + S.dz[cur];
            const uint32_t dw_tmem = tmem + 64u + 64u * static_cast<uint32_t>(l >> 1) + ((l & 1) ? (16u << 16) : 0u);
            // Issue order: dH_l first, then its commit, then dW_l. tcgen05.mma from one thread
            // completes in issue order and a commit covers every earlier MMA, so the epilogue
            // (which needs dH_l) waits on a barrier that does not include dW_l: dW_l runs under
            // this layer's epilogue and is covered by the next layer's commit.
            if (t == 0) {
                umma::fence_after_sync();
                if (l > 0) {
                    const uint32_t id_dh = umma::idesc_bf16(128, di, false, true);
                    for (int kb = 0; kb < dout / 16; ++kb)
                        umma::mma_bf16(tmem, umma::desc_kmajor(dzt, dout, kb),
                                       umma::desc_mnmajor(sbase + S.wt[l], di, kb), id_dh, kb > 0);
                    umma::commit(&bar);
                }
                const uint32_t id_dw = umma::idesc_bf16(64, dout, true, true);
                for (int kb = 0; kb < kRows / 16; ++kb)
                    umma::mma_bf16(dw_tmem, umma::desc_mnmajor(hin, di, kb), umma::desc_mnmajor(dzt, dout, kb), id_dw,
                                   !(first && kb == 0));
                if (l == 0) umma::commit(&bar);  // the tile's last MMAs: wait before the buffers are reused
            }
            // db_l: column sums of dZ_l, 4 row quarters per column, each thread accumulating its
            // own slice across tiles (fixed order; overlaps the MMAs, which only read the tile)
            if (t < kDbSlices * dout) {
                const int c = t % dout, q4 = t / dout;
                const uint8_t* col = smem + S.dz[cur] + umma::tile_offset(0, c, dout);
                float s = 0.0f;
#pragma unroll 8
                for (int rr = 32 * q4; rr < 32 * q4 + 32; ++rr)
                    s += __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(
                        col + (rr >> 3) * (dout * 16) + (rr & 7) * 16));
                dbacc[(q4 * kMaxLayers + l) * kMaxW + c] += s;
            }
            umma::mbar_wait(&bar, phase);
            phase ^= 1;
            umma::fence_after_sync();
            if (l > 0) {
                const int pw = di;  // width of dZ_{l-1}
                for (int c0 = 16 * half; c0 < pw; c0 += 32) {
                    float g[16], y[16];
                    umma::tmem_ld16(tmem + lane_base + c0, g);
                    umma::ld_row8(smem + S.h[l - 1], pw, r, c0, y);
                    umma::ld_row8(smem + S.h[l - 1], pw, r, c0 + 8, y + 8);
                    umma::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) g[j] = a.act == 0 ? g[j] * (1.0f - y[j] * y[j]) : (y[j] > 0.0f ? g[j] : 0.0f);
                    umma::st_row8(smem + S.dz[cur ^ 1], pw, r, c0, g);
                    umma::st_row8(smem + S.dz[cur ^ 1], pw, r, c0 + 8, g + 8);
                }
                umma::fence_async_smem();
                umma::fence_before_sync();
                __syncthreads();
                cur ^= 1;
            }
        }
        first = false;
        umma::fence_before_sync();
        __syncthreads();
    }

    // ---- per-CTA partials: dW from TMEM, db from smem, loss terms
    if (a.mode == 1) {
        umma::fence_after_sync();
        float* part = a.partials + static_cast<int64_t>(blockIdx.x) * a.part_stride;
        for (int l = 0; l < L; ++l) {
            const int dout = n.dout[l], ri = n.rin[l], ro = n.rout[l];
            const int lo = (l & 1) ? 16 : 0;
            const uint32_t col = 64u + 64u * static_cast<uint32_t>(l >> 1);
            for (int c0 = 16 * half; c0 < dout; c0 += 32) {
                float v[16];
                umma::tmem_ld16(tmem + lane_base + col + c0, v);
                umma::tmem_ld_wait();
                const int m = lane - lo;  // dW row (input index) held by this lane
                if (!first && m >= 0 && m < 16) {
                    const int i = m + 16 * quad;
                    if (i < ri)
                        for (int j = 0; j < 16; ++j)
                            if (c0 + j < ro) part[n.woff[l] - n.woff[0] + i * ro + c0 + j] = v[j];
                }
            }
            for (int o = t; o < ro; o += kThreads) {
                float s = 0.0f;
                for (int q4 = 0; q4 < kDbSlices; ++q4) s += dbacc[(q4 * kMaxLayers + l) * kMaxW + o];
                part[n.boff[l] - n.woff[0] + o] = s;
            }
        }
        float* ls = reinterpret_cast<float*>(smem + S.loss);
        for (int off = 16; off > 0; off >>= 1) {
            pl_acc += __shfl_xor_sync(0xffffffffu, pl_acc, off);
            vl_acc += __shfl_xor_sync(0xffffffffu, vl_acc, off);
            en_acc += __shfl_xor_sync(0xffffffffu, en_acc, off);
        }
        if (lane == 0) {
            ls[w * 3 + 0] = pl_acc;
            ls[w * 3 + 1] = vl_acc;
            ls[w * 3 + 2] = en_acc;
        }
        __syncthreads();
        if (t < 3) {
            float s = 0.0f;
            for (int k = 0; k < 8; ++k) s += ls[k * 3 + t];
            a.loss_partials[blockIdx.x * 3 + t] = s;
        }
        if (first) {  // CTA owned no tile: zero its partial slot
            for (int64_t i = t; i < a.part_stride; i += kThreads) part[i] = 0.0f;
        }
    }
    if (t == 0 && a.mode == 0 && a.hsave) umma::bulk_wait_all();  // saved tiles landed in HBM
    umma::fence_before_sync();
    __syncthreads();
    if (w == 0) umma::tmem_free<512>(tmem);
}

// Weight-tile image: exactly the bytes [0, S.x) of k_fast_mlp's shared memory.
__global__ void __launch_bounds__(256) k_build_wimg(const float* __restrict__ params, FastNet n,
                                                    __nv_bfloat16* __restrict__ img) {
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
                                                         int nparts, int64_t Pp, int64_t Pc, float* grads) {
    // 32 parameters per block (lane = parameter, coalesced rows); warp w sums partials
    // w, w+8, ... in order, then the 8 warp sums are added in warp order: a fixed tree.
    __shared__ float ws[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t i = blockIdx.x * 32LL + lane;
    const bool ok = i < Pp + Pc;
    const float* src = !ok ? pp : (i < Pp ? pp + i : pc + (i - Pp));
    const int64_t stride = i < Pp ? Pp : Pc;
    float s = 0.0f;
    if (ok)
        for (int p = w; p < nparts; p += 8) s += src[p * stride];
    ws[w][lane] = s;
    __syncthreads();
    if (w == 0 && ok) {
        float t = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += ws[k][lane];
        grads[i] = t;
    }
}

__global__ void k_reduce_loss(const float* __restrict__ lp, int nparts, int nsets, double ec, float* loss) {
    const int lane = threadIdx.x;
    double pl = 0, vl = 0, en = 0;
    for (int s = 0; s < nsets; ++s)
        for (int p = lane; p < nparts; p += 32) {
            const float* q = lp + (s * nparts + p) * 3;
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
__global__ void __launch_bounds__(256, 4) k_fast_gae(const float* __restrict__ rew, const float* __restrict__ values,
                                                  const float* __restrict__ done_f,
                                                  const float* __restrict__ last_value, int64_t T, int64_t R,
                                                  double gamma, double lam, float* adv, float* ret, bool with_adv,
                                                  double* block_sums) {
    __shared__ double s1[256], s2[256];
    int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    double a1 = 0.0, a2 = 0.0;
    if (s < R) {
        const double gl = gamma * lam;
        const double lv = last_value[s];
        double acc = 0.0, running = lv, next_v = lv;
        for (int64_t hi = T - 1; hi >= 0; hi -= 8) {
            float rr[8], vv[8], dd[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int64_t tt = hi - j;
                if (tt >= 0) {
                    int64_t i = tt * R + s;
                    rr[j] = rew[i];
                    vv[j] = values[i];
                    dd[j] = done_f[i];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
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
size_t fast_mlp_smem_bytes(const FastNet& n) { return carve(n).total; }
size_t fast_wimg_bytes(const FastNet& n) { return carve(n).x; }
size_t fast_hsave_bytes(const FastNet& n) {
    const Smem s = carve(n);
    return n.L > 1 ? s.dz[0] - s.h[0] : 0;
}

void fast_build_wimg(cudaStream_t s, const float* params, const FastNet& n, __nv_bfloat16* img) {
    k_build_wimg<<<148, 256, 0, s>>>(params, n, img);
}

void fast_mlp(cudaStream_t s, const FastLearnArgs& a, int grid) {
    const size_t smem = carve(a.net).total;
    // per-device attribute: set on every launch (cheap, and legal inside stream capture)
    FLW_CUDA(cudaFuncSetAttribute(k_fast_mlp, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    k_fast_mlp<<<grid, kThreads, smem, s>>>(a);
}

void fast_reduce_partials(cudaStream_t s, const float* part_p, const float* part_c, int nparts, int64_t Pp, int64_t Pc,
                          float* grads) {
    k_reduce_partials<<<static_cast<unsigned>((Pp + Pc + 31) / 32), 256, 0, s>>>(part_p, part_c, nparts, Pp, Pc,
                                                                                 grads);
}

void fast_reduce_loss(cudaStream_t s, const float* loss_parts, int nparts, int nsets, double entropy_coef,
                      float* loss) {
    k_reduce_loss<<<1, 32, 0, s>>>(loss_parts, nparts, nsets, entropy_coef, loss);
}

void fast_gae(cudaStream_t s, const float* rew, const float* values, const float* done_f, const float* last_value,
              int64_t TR, int64_t R, double gamma, double lam, float* adv, float* ret, bool with_adv,
              double* block_sums, double* stats) {
    const int nb = static_cast<int>((R + 255) / 256);
    k_fast_gae<<<nb, 256, 0, s>>>(rew, values, done_f, last_value, TR / R, R, gamma, lam, adv, ret, with_adv,
                                  block_sums);
    if (with_adv) k_adv_stats<<<1, 256, 0, s>>>(block_sums, nb, TR, stats);
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
