// Builder-defined environment "synth17x6".
// Test infrastructure: this is the reference-side registration of the builder env,
// written in the reference's EnvSpec/EnvState/StepResult types
// (/root/reference/proj/src/envs/envs.hpp:20-48) and keyed with its counter RNG
// (/root/reference/proj/src/core/rng.hpp:12-38). Only + - * / and comparisons, so the
// dynamics are bit-reproducible in IEEE double on any device with FMA contraction off.
#pragma once
#include <cstdint>

namespace synth {

constexpr int kObs = 17;
constexpr int kAct = 6;
constexpr double kDt = 0.05;
constexpr double kCoupling = 0.3;
constexpr double kDamping = 0.5;
constexpr double kBound = 2.0;
constexpr double kResetLo = -0.1, kResetHi = 0.1;
constexpr uint64_t kTableSeed = 0x73796e;         // "syn"
constexpr uint64_t kResetTag = 0x7265736574;      // same stream tag as envs.cpp:13

}  // namespace synth
