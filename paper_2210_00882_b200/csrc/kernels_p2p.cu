// Gradient all-reduce over NVLink peer memory, fused with the producing reduction and with
// Adam (fast numerics, k GPUs). Replaces  k_reduce_partials -> ncclAllReduce -> k_adam:
//
//   k_reduce_push  grid-stride over 128-parameter chunks: reduces the per-CTA dW partials (fixed
//                  order, float4 rows) and stores the chunk straight into every rank's
//                  inbox[rank] over NVLink, then releases flag[chunk][rank] on each rank (system
//                  scope). The exchange of a chunk overlaps the reduction of the others; it
//                  never waits.
//   k_sum_adam     per chunk (grid-stride) acquires the k flags, sums inbox[0..k-1] in rank order
//                  (every rank computes the identical mean, deterministic), applies Adam and
//                  refreshes the bf16 weight images.
//                  It waits only on k_reduce_push kernels, so no residency requirement.
//
// Flags are monotonically increasing epochs (DeviceCtx::coll_seq), never reset. Region layout
// (identical on every rank, one cudaMalloc, CUDA-IPC exported for one-process-per-GPU runs):
// inbox f32 [2][k][P] (by epoch parity: a fast rank never overwrites data a slow rank has not
// read - it cannot reach exchange e+2 before every rank finished reading exchange e) | grads
// f32 [P] (unused) | flag u64 [chunks][k].
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "engine.hpp"
#include "p2p.cuh"

namespace flw {

namespace {

__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_coll_tick(DeviceCtx* ctx) { ++ctx->coll_seq; }

// Chunks of 128 parameters in the padded index space [policy rows padded to 4][critic rows
// padded to 4] (the learn kernels write 16-byte aligned partial rows), so a lane's float4 never
// straddles the two nets. pad_to_flat maps a padded index to the flat parameter index (-1: pad).
__device__ __forceinline__ int64_t pad_to_flat(const P2pArgs& a, int64_t ip) {
    const int64_t Pps = (a.Pp + 3) / 4 * 4, Pcs = (a.Pc + 3) / 4 * 4;
    if (ip < Pps) return ip < a.Pp ? ip : -1;
    const int64_t c = ip - Pps;
    return c < a.Pc && ip < Pps + Pcs ? a.Pp + c : -1;
}

// A: reduce the per-CTA dW partials of one 128-parameter chunk (fixed order: warp w sums
// partials w, w+8, ... as float4 rows, then the 8 warp sums in warp order) and push the chunk
// into EVERY rank's inbox[rank] over NVLink; then release flag[chunk][rank] on every rank.
// Never waits, so any grid size is safe.
__global__ void __launch_bounds__(256) k_reduce_push(P2pArgs a, int nchunks) {
    __shared__ float4 ws[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint64_t epoch = a.ctx->coll_seq;
    const int64_t P = a.Pp + a.Pc;
    const int64_t Pps = (a.Pp + 3) / 4 * 4, Pcs = (a.Pc + 3) / 4 * 4;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {  // grid-stride over 128-parameter chunks
        const int64_t q0 = 128LL * c + 4 * lane;
        float4 s4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q0 < Pps + Pcs) {
            const bool pol = q0 < Pps;
            const float* base = pol ? a.part_p + q0 : a.part_c + (q0 - Pps);
            const int64_t stride = pol ? Pps : Pcs;
            const int nparts = pol ? a.np : a.nc;
#pragma unroll 4
            for (int p = w; p < nparts; p += 8) {  // loads hoisted, adds in order
                const float4 v = *reinterpret_cast<const float4*>(base + p * stride);
                s4.x += v.x;
                s4.y += v.y;
                s4.z += v.z;
                s4.w += v.w;
            }
        }
        ws[w][lane] = s4;
        __syncthreads();
        if (threadIdx.x < 128) {
            const int64_t i = pad_to_flat(a, 128LL * c + threadIdx.x);
            if (i >= 0) {
                float t = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) t += reinterpret_cast<const float*>(&ws[k][threadIdx.x >> 2])[threadIdx.x & 3];
                for (int r = 0; r < a.k; ++r) {
                    // inbox[epoch & 1]: rank r may still be reading the previous exchange's buffer
                    float* inbox = reinterpret_cast<float*>(a.peers[r] + a.off_inbox) + static_cast<int64_t>(epoch & 1) * a.k * P;
                    inbox[static_cast<int64_t>(a.rank) * P + i] = t;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x < a.k)  // release: the block's chunk stores are ordered before the flag
            st_release_sys(reinterpret_cast<uint64_t*>(a.peers[threadIdx.x] + a.off_sflag) +
                               static_cast<int64_t>(c) * a.k + a.rank,
                           epoch);
    }
}

// B: wait for the k ranks' copies of the chunk, sum them in rank order (every rank computes
// the identical mean) and apply Adam (adam_step, mlp.cpp:146-161; 1/k folded into the step).
// Waits only on A kernels, which never wait: no residency requirement.
__global__ void __launch_bounds__(128) k_sum_adam(P2pArgs a, int nchunks) {
    const uint64_t epoch = a.ctx->coll_seq;
    const int64_t P = a.Pp + a.Pc;
    __shared__ int gave_up;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {  // grid-stride over 128-parameter chunks
        const uint64_t* flag =
            reinterpret_cast<const uint64_t*>(a.peers[a.rank] + a.off_sflag) + static_cast<int64_t>(c) * a.k;
        if (threadIdx.x == 0) gave_up = 0;
        __syncthreads();
        for (int r = threadIdx.x; r < a.k; r += blockDim.x)
            for (uint32_t spin = 1; ld_acquire_sys(flag + r) < epoch; ++spin) {
                // the abort word lives in host memory (a PCIe read): polled every 512 spins only
                if ((spin & 511u) == 0 && *a.abort_flag) {  // the host aborted the group
                    gave_up = 1;
                    break;
                }
                __nanosleep(64);
            }
        __syncthreads();
        if (gave_up) return;
        const int64_t i = pad_to_flat(a, 128LL * c + threadIdx.x);
        if (i >= 0) {
            const float* inbox = reinterpret_cast<const float*>(a.peers[a.rank] + a.off_inbox) +
                                 static_cast<int64_t>(epoch & 1) * a.k * P;
            float gs = 0.0f;
            for (int r = 0; r < a.k; ++r) gs += __ldcv(inbox + static_cast<int64_t>(r) * P + i);
            const double g = __dmul_rn(static_cast<double>(gs), a.gscale);
            const double bc1 = a.ctx->bc1, bc2 = a.ctx->bc2;
            const double mi = __dadd_rn(__dmul_rn(a.b1, a.m[i]), __dmul_rn(__dsub_rn(1.0, a.b1), g));
            const double vi = __dadd_rn(__dmul_rn(a.b2, a.v[i]), __dmul_rn(__dmul_rn(__dsub_rn(1.0, a.b2), g), g));
            a.m[i] = mi;
            a.v[i] = vi;
            const double mhat = __ddiv_rn(mi, bc1), vhat = __ddiv_rn(vi, bc2);
            const double next = __dsub_rn(static_cast<double>(a.params[i]),
                                          __ddiv_rn(__dmul_rn(a.lr, mhat), __dadd_rn(__dsqrt_rn(vhat), a.eps)));
            a.params[i] = static_cast<float>(next);
            if (a.img_p) {  // weight-image entry for the next train iteration's learn kernels
                const bool pol = i < a.Pp;
                const int64_t e = wimg_elem(pol ? a.pol : a.crit, i);
                if (e >= 0) (pol ? a.img_p : a.img_c)[e] = __float2bfloat16(static_cast<float>(next));
            }
        }
        __syncthreads();  // gave_up is rewritten by the next chunk
    }
}

}  // namespace

P2pLayout p2p_layout(int k, int64_t P) {
    P2pLayout L{};
    const int64_t nchunks = (P + 31) / 32;
    auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
    L.off_inbox = 0;
    L.off_grads = al(L.off_inbox + 2 * static_cast<int64_t>(k) * P * 4);  // two parity buffers
    L.off_sflag = al(L.off_grads + P * 4);
    L.off_dflag = al(L.off_sflag + nchunks * k * 8);
    L.bytes = al(L.off_dflag + 8);
    return L;
}

void coll_tick(cudaStream_t s, DeviceCtx* ctx) { k_coll_tick<<<1, 1, 0, s>>>(ctx); }

void reduce_allreduce_adam(cudaStream_t s, const P2pArgs& a) {
    const int64_t padded = (a.Pp + 3) / 4 * 4 + (a.Pc + 3) / 4 * 4;
    const int nchunks = static_cast<int>((padded + 127) / 128);  // <= the layout's flag rows
    const unsigned grid = static_cast<unsigned>(std::min(nchunks, 148 * 8));
    k_reduce_push<<<grid, 256, 0, s>>>(a, nchunks);
    k_sum_adam<<<grid, 128, 0, s>>>(a, nchunks);
}

}  // namespace flw
