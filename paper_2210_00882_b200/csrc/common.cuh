// Shared host/device helpers for the B200 DP-D engine.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "errors.hpp"

namespace flw {

#define FLW_CUDA(x)                                                                                  \
    do {                                                                                             \
        cudaError_t e_ = (x);                                                                        \
        if (e_ != cudaSuccess)                                                                       \
            throw ::flw::Error(::flw::Errc::Runtime,                                                 \
                               std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + __FILE__ + \
                                   ":" + std::to_string(__LINE__));                                  \
    } while (0)

// ------------------------------------------------------------------ counter RNG
// splitmix64 keyed counter generator; same arithmetic as the reference
// (/root/reference/proj/src/core/rng.hpp:12-38), so draws are placement- and device-invariant.
// Host-side progress trace to stderr when FLW_TRACE is set (diagnosing multi-GPU stalls).
inline void flw_trace(const char* what) {
    static const bool on = std::getenv("FLW_TRACE") != nullptr;
    if (on) std::fprintf(stderr, "[flw] %s\n", what);
}

__host__ __device__ __forceinline__ uint64_t rng_mix(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0,
                                                     uint64_t d = 0) {
    uint64_t h = rng_mix(seed);
    h = rng_mix(h ^ a);
    h = rng_mix(h ^ b);
    h = rng_mix(h ^ c);
    h = rng_mix(h ^ d);
    return h;
}

// uniform in [0,1): (k >> 11) * 2^-53 (exact scaling by a power of two).
__host__ __device__ __forceinline__ double rng_uniform(uint64_t k) {
    return static_cast<double>(k >> 11) * (1.0 / 9007199254740992.0);
}

// lo + (hi - lo) * u with every operation individually rounded (no FMA contraction), which is
// what the reference's g++ -O2 x86-64 build computes (rng.hpp:37).
__host__ __device__ __forceinline__ double rng_uniform_range(uint64_t k, double lo, double hi) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), rng_uniform(k)));
#else
    return lo + (hi - lo) * rng_uniform(k);  // host: x86-64 baseline has no FMA to contract into
#endif
}

// Stream separators (interp.cpp:15-17, envs.cpp:13).
constexpr uint64_t kParamStream = 0x706172ULL;
constexpr uint64_t kActionStream = 0x616374ULL;
constexpr uint64_t kEnvStream = 0x656e76ULL;
constexpr uint64_t kResetTag = 0x7265736574ULL;

// Tensor::store for F32 tensors (core/tensor.hpp:74): round the double through float.
__host__ __device__ __forceinline__ double f32r(double v) { return static_cast<double>(static_cast<float>(v)); }

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace flw
