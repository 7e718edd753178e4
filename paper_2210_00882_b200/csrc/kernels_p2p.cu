// Gradient all-reduce over NVLink peer memory, fused with the producing reduction and with
// Adam (fast numerics, k GPUs). Replaces  k_reduce_partials -> ncclAllReduce -> k_adam.
//
// Per 128-parameter chunk: reduce the per-CTA dW partials (fixed order, float4 rows), store the
// chunk straight into every rank's inbox[rank] over NVLink, then (every rank) wait for the k
// copies, sum them in rank order (every rank computes the identical mean, deterministic),
// apply Adam and refresh the bf16 weight images.
//
// Protocol: every inbox entry is ONE 8-byte word {f32 value, u32 epoch} written with a single
// store and polled by the reader until its epoch tag matches (single-copy atomic 64-bit
// accesses: a value can never be seen without its tag) - no release fence or flag round trip
// per chunk (a system-scope release/acquire pair costs microseconds over NVLink). Epochs are
// DeviceCtx::coll_seq (monotonic, never reset). The inbox is double-buffered by epoch parity:
// a fast rank never overwrites data a slow rank has not read - it cannot reach exchange e+2
// before every rank finished reading exchange e.
//
// Two launch forms: k_exchange_adam (one kernel; each block pushes its chunk, then waits for the
// same chunk from the other ranks) when every peer is another GPU, else k_reduce_push +
// k_sum_adam (the first never waits, so co-located ranks cannot fill a device with waiting
// blocks). Region layout (identical on every rank, one cudaMalloc, CUDA-IPC exported for one-
// process-per-GPU runs): inbox u32x2 [2][k][Ptot] | grads f32 [P] (unused) | flag u64 (unused).
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "engine.hpp"
#include "p2p.cuh"

namespace flw {

namespace {

__device__ __forceinline__ void st_tagged(uint2* p, float v, uint32_t epoch) {
    asm volatile("st.relaxed.sys.global.v2.u32 [%0], {%1, %2};\n" ::"l"(p), "r"(__float_as_uint(v)), "r"(epoch)
                 : "memory");
}

__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;\n" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];\n" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint2 ld_tagged(const uint2* p) {
    uint2 v;
    asm volatile("ld.relaxed.sys.global.v2.u32 {%0, %1}, [%2];\n" : "=r"(v.x), "=r"(v.y) : "l"(p) : "memory");
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

// Reduce the per-CTA dW partials of one 128-parameter chunk (fixed order: warp w sums partials
// w, w+8, ... as float4 rows, then the 8 warp sums in warp order) and push the chunk into EVERY
// rank's inbox[rank] over NVLink; then release flag[chunk][rank] on every rank. 256 threads.
__device__ __forceinline__ void reduce_push_chunk(const P2pArgs& a, int c, uint64_t epoch, float4 (*ws)[32]) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t P = a.Pp + a.Pc;
    const int64_t Pps = (a.Pp + 3) / 4 * 4, Pcs = (a.Pc + 3) / 4 * 4;
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
                // (the inbox is laid out over ALL parameters: a launch over one net writes its
                // own columns [off, off + P), never another launch's)
                uint2* inbox = reinterpret_cast<uint2*>(a.peers[r] + a.off_inbox) + static_cast<int64_t>(epoch & 1) * a.k * a.Ptot;
                st_tagged(inbox + static_cast<int64_t>(a.rank) * a.Ptot + a.off + i, t, static_cast<uint32_t>(epoch));
            }
        }
    }
    // a per-(chunk, rank) hint word after the chunk's data: the readers poll this one word
    // instead of the chunk's 128 x k tagged words (which they still check afterwards - the
    // hint carries no ordering, so no fence is needed here)
    __syncthreads();
    if (threadIdx.x < a.k)
        st_relaxed_u64(reinterpret_cast<uint64_t*>(a.peers[threadIdx.x] + a.off_sflag) +
                           (static_cast<int64_t>(a.flag0) + c) * a.k + a.rank,
                       epoch);
}

// Wait (the whole block) until the k ranks' copies of chunk c carry this exchange's epoch tag.
// One warp polls: lane l checks the chunk's words l, l+32, ... of every rank, resuming at the
// first word it has not seen tagged yet; lane 0 alone reads the host-mapped abort word (a PCIe
// read), every 64 rounds - one poller per block keeps a long wait off the PCIe bus. false: the
// host aborted the group.
__device__ __forceinline__ bool wait_chunk(const P2pArgs& a, int c, uint64_t epoch, int* s_abort) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        const int64_t P = a.Pp + a.Pc;
        const uint2* inbox = reinterpret_cast<const uint2*>(a.peers[a.rank] + a.off_inbox) +
                             static_cast<int64_t>(epoch & 1) * a.k * a.Ptot + a.off;
        const uint32_t tag = static_cast<uint32_t>(epoch);
        int ab = 0;
        // phase 1: the k hint words of this chunk (lane r: rank r), with a growing back-off -
        // a long wait must not flood this GPU's L2 (the peers' NVLink stores land there)
        const uint64_t* hint = reinterpret_cast<const uint64_t*>(a.peers[a.rank] + a.off_sflag) +
                               (static_cast<int64_t>(a.flag0) + c) * a.k;
        uint32_t ns = 32;
        for (uint32_t round = 1;; ++round) {
            const bool here = lane >= a.k || ld_relaxed_u64(hint + lane) >= epoch;
            if (__all_sync(0xffffffffu, here)) break;
            if ((round & 255u) == 0) {
                ab = __shfl_sync(0xffffffffu, lane == 0 ? static_cast<int>(*a.abort_flag) : 0, 0);
                if (ab) break;
            }
            __nanosleep(ns);
            ns = ns < 1024u ? 2u * ns : 1024u;
        }
        // phase 2: every word of the chunk carries the epoch's tag (normally already true)
        int pos = 0;  // next (rank, word) of this lane to check: rank = pos / 4, word = lane + 32 (pos % 4)
        for (uint32_t round = 1; !ab; ++round) {
            for (; pos < 4 * a.k; ++pos) {
                const int64_t i = pad_to_flat(a, 128LL * c + lane + 32 * (pos & 3));
                if (i >= 0 && ld_tagged(inbox + static_cast<int64_t>(pos >> 2) * a.Ptot + i).y != tag) break;
            }
            if (__all_sync(0xffffffffu, pos == 4 * a.k)) break;
            if ((round & 63u) == 0) {
                ab = __shfl_sync(0xffffffffu, lane == 0 ? static_cast<int>(*a.abort_flag) : 0, 0);
                if (ab) break;
            }
            __nanosleep(100);
        }
        if (lane == 0) *s_abort = ab;
    }
    __syncthreads();
    return *s_abort == 0;
}

// Sum the k copies of this thread's parameter (threads [0, 128) of the block; wait_chunk saw
// them tagged) in rank order - every rank computes the identical mean - and apply Adam
// (adam_step, mlp.cpp:146-161; 1/k folded into the step).
__device__ __forceinline__ void sum_adam_chunk(const P2pArgs& a, int c, uint64_t epoch) {
    const int64_t P = a.Pp + a.Pc;
    const int64_t il = threadIdx.x < 128 ? pad_to_flat(a, 128LL * c + threadIdx.x) : -1;  // this launch's index
    if (il < 0) return;
    const int64_t i = a.off + il;  // flat parameter index
    const uint2* inbox = reinterpret_cast<const uint2*>(a.peers[a.rank] + a.off_inbox) +
                         static_cast<int64_t>(epoch & 1) * a.k * a.Ptot + a.off;
    float gs = 0.0f;
    for (int r = 0; r < a.k; ++r) gs += __uint_as_float(ld_tagged(inbox + static_cast<int64_t>(r) * a.Ptot + il).x);
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
        const bool pol = !a.critic_only && il < a.Pp;
        const int64_t e = wimg_elem(pol ? a.pol : a.crit, i);
        if (e >= 0) (pol ? a.img_p : a.img_c)[e] = __float2bfloat16(static_cast<float>(next));
    }
}

// A (two-kernel form): reduce + push of every chunk; never waits, so any grid size is safe.
__global__ void __launch_bounds__(256) k_reduce_push(P2pArgs a, int nchunks) {
    __shared__ float4 ws[8][32];
    const uint64_t epoch = a.ctx->coll_seq;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {  // grid-stride over 128-parameter chunks
        reduce_push_chunk(a, c, epoch, ws);
        __syncthreads();  // ws is rewritten by the next chunk
    }
}

// B (two-kernel form): per chunk, wait for the k copies, sum, Adam. Waits only on A kernels,
// which never wait: no residency requirement.
__global__ void __launch_bounds__(256) k_sum_adam(P2pArgs a, int nchunks) {
    __shared__ int s_abort;
    const uint64_t epoch = a.ctx->coll_seq;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        if (!wait_chunk(a, c, epoch, &s_abort)) return;
        sum_adam_chunk(a, c, epoch);
        __syncthreads();  // s_abort is rewritten by the next chunk
    }
}

// Fused form (peers on distinct GPUs): each block reduces and pushes its chunk, then waits for
// the same chunk from the other ranks and applies Adam - one launch, and a chunk's exchange
// overlaps the reduction of the others. A block waits only for the block of the same index on
// the other ranks, which runs the same chunk sequence (grid-stride, grid <= the co-resident
// capacity, checked by the host): every block is eventually resident, no cyclic wait.
__global__ void __launch_bounds__(256) k_exchange_adam(P2pArgs a, int nchunks) {
    __shared__ float4 ws[8][32];
    __shared__ int s_abort;
    const uint64_t epoch = a.ctx->coll_seq;
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
        reduce_push_chunk(a, c, epoch, ws);
        if (!wait_chunk(a, c, epoch, &s_abort)) return;
        sum_adam_chunk(a, c, epoch);
        __syncthreads();  // ws / s_abort are rewritten by the next chunk
    }
}

}  // namespace

P2pLayout p2p_layout(int k, int64_t P) {
    P2pLayout L{};
    const int64_t nchunks = (P + 31) / 32;
    auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
    L.off_inbox = 0;
    L.off_grads = al(L.off_inbox + 2 * static_cast<int64_t>(k) * P * 8);  // two parity buffers of tagged words
    L.off_sflag = al(L.off_grads + P * 4);
    L.off_dflag = al(L.off_sflag + nchunks * k * 8);
    L.bytes = al(L.off_dflag + 8);
    return L;
}

void coll_tick(cudaStream_t s, DeviceCtx* ctx) { k_coll_tick<<<1, 1, 0, s>>>(ctx); }

void reduce_allreduce_adam(cudaStream_t s, const P2pArgs& a, bool fused) {
    const int64_t padded = (a.Pp + 3) / 4 * 4 + (a.Pc + 3) / 4 * 4;
    const int nchunks = static_cast<int>((padded + 127) / 128);  // <= the layout's flag rows
    if (fused) {
        // grid <= the blocks that can be resident at once (the fused kernel's blocks wait)
        int dev = 0, sms = 0, per_sm = 0;
        FLW_CUDA(cudaGetDevice(&dev));
        FLW_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        FLW_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_exchange_adam, 256, 0));
        const int cap = std::max(1, sms * per_sm);
        k_exchange_adam<<<static_cast<unsigned>(std::min(nchunks, cap)), 256, 0, s>>>(a, nchunks);
        return;
    }
    const unsigned grid = static_cast<unsigned>(std::min(nchunks, 148 * 8));
    k_reduce_push<<<grid, 256, 0, s>>>(a, nchunks);
    k_sum_adam<<<grid, 256, 0, s>>>(a, nchunks);
}

}  // namespace flw
