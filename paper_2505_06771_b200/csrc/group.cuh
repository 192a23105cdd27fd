// group.cuh — lockstep sub-warp groups.
//
// A warp holds 32/L environments, L lanes each (lane r = robot r). All 32
// lanes execute every instruction of the step in lockstep: every loop bound
// that contains a collective is warp-uniform and per-environment decisions
// are predicates, so every shuffle / vote uses the full mask (no WARPSYNC,
// no divergent re-convergence). Reductions run over the L lanes of a group
// (shuffle `width` = L).
#pragma once

#include <cuda_runtime.h>

namespace mrsim_dev {

template <int L>
struct Grp {
    static_assert(L == 4 || L == 8 || L == 16, "group width");
    static constexpr unsigned kFull = 0xffffffffu;
    int lane;  // 0..L-1 within the group
    __device__ __forceinline__ Grp() : lane(static_cast<int>(threadIdx.x) & (L - 1)) {}
    __device__ __forceinline__ static unsigned group_bits() {
        return ((L == 32) ? 0xffffffffu : ((1u << L) - 1u)) << ((threadIdx.x & 31) & ~(L - 1));
    }
    __device__ __forceinline__ static void sync() { __syncwarp(kFull); }
    template <class T>
    __device__ __forceinline__ T shfl(T v, int src) const { return __shfl_sync(kFull, v, src, L); }
    template <class T>
    __device__ __forceinline__ T sum(T v) const {
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o, L);
        return v;
    }
    template <class T>
    __device__ __forceinline__ T min(T v) const {
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
            const T w = __shfl_xor_sync(kFull, v, o, L);
            v = w < v ? w : v;
        }
        return v;
    }
    // any over this group's lanes
    __device__ __forceinline__ bool any(bool p) const { return (__ballot_sync(kFull, p) & group_bits()) != 0u; }
    // lowest lane of this group with p set, or -1
    __device__ __forceinline__ int first(bool p) const {
        const unsigned b = (__ballot_sync(kFull, p) & group_bits()) >> ((threadIdx.x & 31) & ~(L - 1));
        return b ? __ffs(b) - 1 : -1;
    }
    // warp-wide (all groups) votes / reductions, for warp-uniform loop bounds
    __device__ __forceinline__ static bool warp_any(bool p) { return __any_sync(kFull, p); }
    __device__ __forceinline__ static int warp_max(int v) { return __reduce_max_sync(kFull, v); }
    // argmax with ties to the lowest index (first-maximal `v > worst` scans, qp.hpp:228-238);
    // idx < 0 = none
    // idx < 0 (none) travels as kNone so it loses every tie; callers pass v =
    // the scan threshold (argmax) / +inf (argmin) with it, which any real
    // candidate beats strictly.
    static constexpr int kNone = 0x7fffffff;
    template <class T>
    __device__ __forceinline__ void argmax(T& v, int& idx) const {
        idx = idx < 0 ? kNone : idx;
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
            const T ov = __shfl_xor_sync(kFull, v, o, L);
            const int oi = __shfl_xor_sync(kFull, idx, o, L);
            const bool take = (ov > v) | ((ov == v) & (oi < idx));  // no short-circuit: no branch
            v = take ? ov : v;
            idx = take ? oi : idx;
        }
        idx = idx == kNone ? -1 : idx;
    }
    // argmin with ties to the lowest index (`t < t1`, qp.hpp:294-302)
    template <class T>
    __device__ __forceinline__ void argmin(T& v, int& idx) const {
        idx = idx < 0 ? kNone : idx;
#pragma unroll
        for (int o = L / 2; o > 0; o >>= 1) {
            const T ov = __shfl_xor_sync(kFull, v, o, L);
            const int oi = __shfl_xor_sync(kFull, idx, o, L);
            const bool take = (ov < v) | ((ov == v) & (oi < idx));
            v = take ? ov : v;
            idx = take ? oi : idx;
        }
        idx = idx == kNone ? -1 : idx;
    }
};

}  // namespace mrsim_dev
