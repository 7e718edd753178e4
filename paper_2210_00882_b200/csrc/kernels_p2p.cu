// Gradient all-reduce over NVLink peer memory, fused with the producing reduction and with
// Adam (fast numerics, k GPUs). Replaces  k_reduce_partials -> ncclAllReduce -> k_adam:
//
//   k_reduce_push  one block per 32-parameter chunk reduces the per-CTA dW partials (fixed
//                  order) and its warp r stores the chunk straight into rank r's inbox[rank]
//                  over NVLink, then releases flag[chunk][rank] on rank r (system scope). The
//                  exchange of a chunk overlaps the reduction of the others; it never waits.
//   k_sum_adam     one warp per chunk acquires the k flags, sums inbox[0..k-1] in rank order
//                  (every rank computes the identical mean, deterministic) and applies Adam.
//                  It waits only on k_reduce_push kernels, so no residency requirement.
//
// Flags are monotonically increasing epochs (DeviceCtx::coll_seq), never reset. Region layout
// (identical on every rank, one cudaMalloc, CUDA-IPC exported for one-process-per-GPU runs):
// inbox f32 [2][k][P] (by epoch parity: a fast rank never overwrites data a slow rank has not
// read - it cannot reach exchange e+2 before every rank finished reading exchange e) | grads
// f32 [P] (unused) | flag u64 [chunks][k].
#include <cuda_runtime.h>

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

// A: reduce the per-CTA dW partials of one 32-parameter chunk (fixed order) and push the chunk
// into EVERY rank's inbox[rank] over NVLink; then release flag[chunk][rank] on every rank.
// Never waits, so any grid size is safe.
__global__ void __launch_bounds__(256) k_reduce_push(P2pArgs a) {
    __shared__ float ws[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int c = blockIdx.x;
    const uint64_t epoch = a.ctx->coll_seq;
    const int64_t P = a.Pp + a.Pc;
    const int64_t i = 32LL * c + lane;
    const bool ok = i < P;
    const float* src = !ok ? a.part_p : (i < a.Pp ? a.part_p + i : a.part_c + (i - a.Pp));
    const int64_t stride = i < a.Pp ? a.Pp : a.Pc;
    const int nparts = i < a.Pp ? a.np : a.nc;
    float s = 0.0f;
    if (ok) {
#pragma unroll 8
        for (int p = w; p < nparts; p += 8) s += src[p * stride];  // loads hoisted, adds in order
    }
    ws[w][lane] = s;
    __syncthreads();
    float t = 0.0f;
#pragma unroll
    for (int k = 0; k < 8; ++k) t += ws[k][lane];
    for (int r = w; r < a.k; r += 8) {  // warp w pushes the chunk to ranks w, w+8, ...
        // inbox[epoch & 1]: rank r may still be reading the previous exchange's buffer
        float* inbox = reinterpret_cast<float*>(a.peers[r] + a.off_inbox) + static_cast<int64_t>(epoch & 1) * a.k * P;
        if (ok) inbox[static_cast<int64_t>(a.rank) * P + i] = t;
        __syncwarp();
        if (lane == 0)  // release: this warp's chunk stores are ordered before the flag
            st_release_sys(reinterpret_cast<uint64_t*>(a.peers[r] + a.off_sflag) +
                               static_cast<int64_t>(c) * a.k + a.rank,
                           epoch);
    }
}

// B: wait for the k ranks' copies of the chunk, sum them in rank order (every rank computes
// the identical mean) and apply Adam (adam_step, mlp.cpp:480-495; 1/k folded into the step).
// Waits only on A kernels, which never wait: no residency requirement.
__global__ void __launch_bounds__(32) k_sum_adam(P2pArgs a) {
    const int lane = threadIdx.x;
    const int c = blockIdx.x;
    const uint64_t epoch = a.ctx->coll_seq;
    const int64_t P = a.Pp + a.Pc;
    const uint64_t* flag = reinterpret_cast<const uint64_t*>(a.peers[a.rank] + a.off_sflag) + static_cast<int64_t>(c) * a.k;
    for (int r = lane; r < a.k; r += 32)
        while (ld_acquire_sys(flag + r) < epoch) __nanosleep(32);
    __syncwarp();
    const int64_t i = 32LL * c + lane;
    if (i >= P) return;
    const float* inbox =
        reinterpret_cast<const float*>(a.peers[a.rank] + a.off_inbox) + static_cast<int64_t>(epoch & 1) * a.k * P;
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
    const unsigned nchunks = static_cast<unsigned>((a.Pp + a.Pc + 31) / 32);
    k_reduce_push<<<nchunks, 256, 0, s>>>(a);
    k_sum_adam<<<nchunks, 32, 0, s>>>(a);
}

}  // namespace flw
