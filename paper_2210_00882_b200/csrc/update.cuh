// The fused per-iteration parameter update (k_reduce_adam) as device functions: the fixed-order
// partial sums of k_reduce_partials and Adam with double moments (mlp.cpp:146-161, as k_adam),
// plus the bf16 weight-image entry of every weight.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "engine.hpp"
#include "fast.cuh"

namespace flw {

// Adam step t of this update and its bias corrections (k_adam_tick's values, not yet stored)
__device__ __forceinline__ void adam_step_consts(const FastUpdateArgs& a, int64_t& t, double& bc1, double& bc2) {
    t = a.ctx->adam_t + 1;
    bc1 = t <= a.bc_len ? a.bc_table[t - 1].x : 1.0 - pow(0.9, static_cast<double>(t));
    bc2 = t <= a.bc_len ? a.bc_table[t - 1].y : 1.0 - pow(0.999, static_cast<double>(t));
}

// One 128-parameter chunk c, run by 256 threads (tid 0..255, sync() a barrier over exactly
// them). Padded index space [policy rows padded to Pps][critic rows padded to Pcs], so a lane's
// float4 never straddles the two nets. Lane -> 4 consecutive parameters; warp w sums partial
// slots w, w+8, ... in order, then the 8 warp sums are added in warp order (per parameter); Adam
// then runs one parameter per thread (tid < 128). The Adam operands and the weight-image index
// are fetched before the sums, and each warp issues up to kBatch partial loads before its first
// add (the chunk is a chain of memory round trips, not a bandwidth problem at C2 sizes).
template <int kBatch = 12, bool kPdl = false, class Sync>
__device__ __forceinline__ void update_chunk(const FastUpdateArgs& a, int64_t c, int tid, float4 (*ws)[32],
                                             double bc1, double bc2, Sync sync) {
    const int lane = tid & 31, w = tid >> 5;
    const int64_t Pps = (a.Pp + 3) / 4 * 4, Pcs = (a.Pc + 3) / 4 * 4;
    const int ln = (tid & 127) >> 2, j = tid & 3;
    const int64_t ipad = c * 128LL + (tid & 127);
    const bool inpol = ipad < Pps;
    const int64_t i = a.off + (inpol ? ipad : a.Pp + (ipad - Pps));  // flat parameter index
    const bool mine = tid < 128 && (inpol ? ipad < a.Pp : (ipad - Pps < a.Pc && ipad < Pps + Pcs));
    double m0 = 0.0, v0 = 0.0;
    float p0 = 0.0f;
    int64_t e = -1;
    bool ip = false;
    if (mine) {
        m0 = a.m[i];
        v0 = a.v[i];
        p0 = a.params[i];
        ip = !a.critic_only && i < a.Pp;
        e = wimg_elem(ip ? a.pol : a.crit, i);
    }
    // programmatic dependent launch: everything above is the previous iteration's state; the
    // partial slots below are the learn kernel's output
    if constexpr (kPdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t q0 = c * 128LL + 4 * lane;  // first of this lane's 4 padded indices
    float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (q0 < Pps + Pcs) {
        const bool pol = q0 < Pps;
        const float* base = pol ? a.pp + q0 : a.pc + (q0 - Pps);
        const int64_t stride = pol ? Pps : Pcs;
        const int nparts = pol ? a.np : a.nc;
        for (int pw = w; pw < nparts; pw += 8 * kBatch) {
            float4 buf[kBatch];
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
                const int p = pw + 8 * k;
                buf[k] = p < nparts ? __ldcg(reinterpret_cast<const float4*>(base + p * stride))
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int k = 0; k < kBatch; ++k) {
                if (pw + 8 * k < nparts) {
                    s4.x += buf[k].x;
                    s4.y += buf[k].y;
                    s4.z += buf[k].z;
                    s4.w += buf[k].w;
                }
            }
        }
    }
    ws[w][lane] = s4;
    sync();
    if (mine) {
        float gsum = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) gsum += reinterpret_cast<const float*>(&ws[k][ln])[j];
        a.grads[i] = gsum;
        const double g = static_cast<double>(gsum);
        const double mi = __dadd_rn(__dmul_rn(a.b1, m0), __dmul_rn(__dsub_rn(1.0, a.b1), g));
        const double vi = __dadd_rn(__dmul_rn(a.b2, v0), __dmul_rn(__dmul_rn(__dsub_rn(1.0, a.b2), g), g));
        a.m[i] = mi;
        a.v[i] = vi;
        const double mhat = __ddiv_rn(mi, bc1), vhat = __ddiv_rn(vi, bc2);
        const float next = static_cast<float>(
            __dsub_rn(static_cast<double>(p0), __ddiv_rn(__dmul_rn(a.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), a.eps))));
        a.params[i] = next;
        // weight-image entry (biases are read from params by the learn kernels)
        if (e >= 0) (ip ? a.img_p : a.img_c)[e] = __float2bfloat16(next);
    }
    sync();  // ws is rewritten by the next chunk
}

__host__ __device__ inline int update_chunks(const FastUpdateArgs& a) {
    return static_cast<int>(((a.Pp + 3) / 4 * 4 + (a.Pc + 3) / 4 * 4 + 127) / 128);
}

// After this block's chunks: one arrival on a.counter; the arrival that completes a.arrivals
// advances the Adam step counter (when a.advance) and re-arms the counter. Every arriving block
// has read the old counter before it arrives. Call from one thread.
__device__ __forceinline__ void update_arrive(const FastUpdateArgs& a, int64_t t, double bc1, double bc2,
                                              unsigned arrivals) {
    __threadfence();
    if (atomicAdd(a.counter, 1u) == arrivals - 1) {
        if (a.advance) {
            a.ctx->adam_t = t;
            a.ctx->bc1 = bc1;
            a.ctx->bc2 = bc2;
        }
        *a.counter = 0u;
    }
}

}  // namespace flw
