// Gradient exchange over NVLink peer memory (kernels_p2p.cu): the fused
// reduce -> all-reduce -> Adam step of fast numerics on k GPUs.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "fast.cuh"

namespace flw {

struct DeviceCtx;

struct P2pLayout {  // byte offsets inside every rank's exchange region
    int64_t off_inbox, off_grads, off_sflag, off_dflag, bytes;
};
P2pLayout p2p_layout(int k, int64_t P);

struct P2pArgs {
    const float* part_p;  // [nparts, Pp] per-CTA dW partials of the policy net
    const float* part_c;  // [nparts, Pc] ... of the critic
    int np, nc;  // partial slots written by the policy / critic learn launches
    int64_t Pp, Pc;
    int rank, k;
    uint8_t* const* peers;  // device array [k]: every rank's exchange region, mapped here
    int64_t off_inbox, off_grads, off_sflag, off_dflag;
    const DeviceCtx* ctx;   // coll_seq (epoch), Adam bias corrections
    // host-mapped abort word: nonzero makes every flag wait give up (a peer failed or the host's
    // deadline passed); the update is then skipped and the host reports Timeout / PeerFailure
    const volatile unsigned* abort_flag;
    float* params;
    double *m, *v;
    double lr, b1, b2, eps, gscale;
    // optional: also refresh the bf16 weight-tile images (null: the next learn rebuilds them)
    FastNet pol, crit;
    __nv_bfloat16 *img_p, *img_c;
    // one net only (see FastUpdateArgs): flat offset of its first parameter, critic rows;
    // Ptot = all parameters (the inbox layout, identical for every launch)
    int64_t off = 0, Ptot = 0;
    int flag0 = 0;  // first hint-word row of this launch's chunks (launches of one net: disjoint rows)
    bool critic_only = false;
};

void coll_tick(cudaStream_t s, DeviceCtx* ctx);  // ++ctx->coll_seq (one per exchange)
// fused: one kernel (reduce + push + wait + Adam per chunk); only when every peer region lives
// on another GPU (blocks of co-located ranks could fill the device and wait on each other)
void reduce_allreduce_adam(cudaStream_t s, const P2pArgs& a, bool fused);

}  // namespace flw
