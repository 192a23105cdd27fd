// mrsim_device.cuh — device-side building blocks shared by every kernel:
// the flattened per-launch parameter block, the counter-based SplitMix64
// RNG (bit-exact with rng.hpp), sub-warp group collectives, and small
// math helpers templated on the compute precision.
//
// Reference paths below are relative to /root/reference/proj/include/mrsim.
#pragma once

// Dynamic work distribution in the persistent kernels (step, scripted planner): warps take
// their next task from a per-launch counter instead of a static grid stride (A/B switch).
#ifndef MRSIM_DYN_SCHED
#define MRSIM_DYN_SCHED 1
#endif

#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "mrsim_cuda.h"

// Device bounds checks (builds with -DMRSIM_DEVICE_CHECKS only; scripts/device_checks.sh): the
// substitute for compute-sanitizer, which this GPU pool refuses. Index asserts at the shared
// accessors, guard words between every shared-memory sub-array of a group (filled per task and
// verified at its end) and guard tails behind the context's device allocations. A failed check
// prints its site and traps, so the launch fails and every test using it fails loudly.
#ifdef MRSIM_DEVICE_CHECKS
#define MRSIM_DCHECK(cond)                                                                              \
    do {                                                                                                \
        if (!(cond)) {                                                                                  \
            printf("MRSIM_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,  \
                   static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                        \
            __trap();                                                                                   \
        }                                                                                               \
    } while (0)
#define MRSIM_GUARD_WORDS 4  // 16-byte guard between shared sub-arrays
#else
#define MRSIM_DCHECK(cond) \
    do {                   \
    } while (0)
#define MRSIM_GUARD_WORDS 0
#endif
constexpr unsigned kGuardPattern = 0xA5C3E10Fu;

namespace mrsim_dev {

// ---------------------------------------------------------------------------
// Precision traits. fp64 mirrors the reference's tolerances exactly
// (qp.hpp:183 tolerance 1e-9, qp.hpp:71/115/248/304 pivots 1e-14, 295 r>1e-12);
// fp32 scales them to its unit roundoff (rows are unit-norm, |u| <= 0.48).
// ---------------------------------------------------------------------------
template <class Real>
struct Prec;
template <>
struct Prec<float> {
    static constexpr float tol = 2e-6f;       // accepted constraint violation
    static constexpr float eps_z = 1e-10f;    // |z|^2 below which the new normal is dependent
    static constexpr float eps_r = 1e-6f;     // r_a > eps_r counts as a blocking multiplier
    static constexpr float eps_row = 1e-14f;  // zero-row threshold of fold_rows
};
template <>
struct Prec<double> {
    static constexpr double tol = 1e-9;
    static constexpr double eps_z = 1e-14;
    static constexpr double eps_r = 1e-12;
    static constexpr double eps_row = 1e-14;
};

__device__ __forceinline__ float dsqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double dsqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float dhypot(float a, float b) { return hypotf(a, b); }
__device__ __forceinline__ double dhypot(double a, double b) { return hypot(a, b); }
__device__ __forceinline__ void dsincos(float x, float* s, float* c) { sincosf(x, s, c); }
__device__ __forceinline__ void dsincos(double x, double* s, double* c) { sincos(x, s, c); }
__device__ __forceinline__ float dabs(float x) { return fabsf(x); }
__device__ __forceinline__ double dabs(double x) { return fabs(x); }
template <class T>
__device__ __forceinline__ T dmin(T a, T b) { return a < b ? a : b; }
template <class T>
__device__ __forceinline__ T dmax(T a, T b) { return a > b ? a : b; }
// core.hpp:144 clamp(v, lo, hi) = min(max(v, lo), hi)
template <class T>
__device__ __forceinline__ T dclamp(T v, T lo, T hi) { return dmin(dmax(v, lo), hi); }

template <class Real>
struct Consts;
template <>
struct Consts<float> {
    static constexpr float pi = 3.14159265358979323846f;
    static constexpr float two_pi = 6.28318530717958647692f;
    static constexpr float inf = __builtin_huge_valf();
};
template <>
struct Consts<double> {
    static constexpr double pi = 3.14159265358979323846;
    static constexpr double two_pi = 6.28318530717958647692;
    static constexpr double inf = __builtin_huge_val();
};

// ---------------------------------------------------------------------------
// SplitMix64 counter RNG (rng.hpp:15-67). Pure integer math => bit-exact.
// ---------------------------------------------------------------------------
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t kForkSalt = 0x632BE59BD9B4E019ULL;
constexpr uint64_t kEpisodeTag = 0xE915E915E915E915ULL;  // harness.hpp:22
constexpr uint64_t kPolicyTag = 0x9D0C7E5F00000001ULL;   // harness.hpp:23

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {  // rng.hpp:17-21
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t key_from_seed(uint64_t seed) {  // rng.hpp:29-31
    return mix64(seed + kGamma);
}
__host__ __device__ __forceinline__ uint64_t fork_key(uint64_t key, uint64_t tag) {  // rng.hpp:35-37
    return mix64(key ^ mix64(tag * kGamma + kForkSalt));
}
// harness.hpp:25-27
__host__ __device__ __forceinline__ uint64_t derive_episode_seed(uint64_t root, int64_t episode) {
    return fork_key(fork_key(key_from_seed(root), kEpisodeTag),
                    static_cast<uint64_t>(static_cast<int>(episode)));
}

struct Rng {  // SplitRng{key, ctr} (rng.hpp:25-67)
    uint64_t key;
    uint64_t ctr;
    __device__ __forceinline__ uint64_t next_u64() {  // rng.hpp:39-42
        ++ctr;
        return mix64(key + ctr * kGamma);
    }
    __device__ __forceinline__ double uniform() {  // rng.hpp:45-47
        return static_cast<double>(next_u64() >> 11) * 0x1.0p-53;
    }
    // lo + (hi - lo) * u with the reference's two roundings (no FMA contraction)
    __device__ __forceinline__ double uniform(double lo, double hi) {
        return __dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), uniform()));
    }
    __device__ __forceinline__ uint64_t uniform_int(uint64_t n) {  // rng.hpp:52-55 (128-bit mulhi)
        return __umul64hi(next_u64(), n);
    }
    __device__ __forceinline__ double normal() {  // rng.hpp:59-64
        double u1 = uniform();
        double u2 = uniform();
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
    }
};

// policy_stream(seed, step, robot).uniform_int(5) (harness.hpp:29-34, policy.hpp:448-449),
// with the per-episode prefix from_seed(seed).fork(kPolicyTag) precomputed.
__device__ __forceinline__ int policy_action(uint64_t policy_key, int step, int robot) {
    uint64_t k = fork_key(fork_key(policy_key, static_cast<uint64_t>(step)), static_cast<uint64_t>(robot));
    return static_cast<int>(__umul64hi(mix64(k + kGamma), 5ULL));
}
__host__ __device__ __forceinline__ uint64_t policy_key_of(uint64_t seed) {
    return fork_key(key_from_seed(seed), kPolicyTag);
}

// ---------------------------------------------------------------------------
// Device error word, ordered like the reference's step_batch: validate_actions
// checks every env's actions before any env is stepped (batch.hpp:226-237,
// 271), so an invalid action anywhere outranks a physics/spawn error in any
// env; within a class the lowest env wins (the sequential order).
// Layout (u64, atomicMin): [class:1][env:39][robot:8][detail:8][code:8],
// class 0 = invalid action, 1 = every other error.
// ---------------------------------------------------------------------------
enum DevErr : unsigned {
    kErrInvalidAction = 1,   // invalid_argument: step_batch: invalid action
    kErrCoincident = 2,      // domain_error: coincident robot positions
    kErrNonFinite = 3,       // domain_error: wrap_angle non-finite
    kErrSpawn = 4,           // runtime_error: sample_poses could not place robot
    kErrGoals = 5,           // runtime_error: navigation could not place goals
    kErrPrey = 6,            // runtime_error: predator_prey could not place prey
};
constexpr int kErrEnvBits = 39;
__device__ __forceinline__ void report_error(unsigned long long* err, long long env, int robot, unsigned code,
                                             int detail = 0) {
    const unsigned long long cls = code == kErrInvalidAction ? 0ull : 1ull;
    unsigned long long v = (cls << 63) |
                           ((static_cast<unsigned long long>(env) & ((1ull << kErrEnvBits) - 1)) << 24) |
                           (static_cast<unsigned long long>(robot & 0xff) << 16) |
                           (static_cast<unsigned long long>(detail & 0xff) << 8) | (code & 0xff);
    atomicMin(err, v);
}

}  // namespace mrsim_dev
