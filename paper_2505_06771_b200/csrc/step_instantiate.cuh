// step_instantiate.cuh — included by step_<task>.cu with MRSIM_TASK_ID set:
// instantiates the fused step kernel for the three group widths and both
// precisions, and the reset kernel.
#pragma once

#include <type_traits>

#include "launch.h"

namespace mrsim_host {

template <class Real, int L, int MP, int MO>
static cudaError_t launch_V(const mrsim_dev::StepParams<Real>& p, int grid, int block, int smem, cudaStream_t stream) {
    auto k = mrsim_dev::step_kernel<Real, L, MP, MO, MRSIM_TASK_ID, false>;
    static int opted[2][16] = {};  // dynamic shared memory already opted in, per instantiation and device
    int multi = 0;
    if constexpr (std::is_same_v<Real, double>) {  // mrsim_rollout (fp64 product path only)
        if (p.n_steps > 1) {
            k = mrsim_dev::step_kernel<Real, L, MP, MO, MRSIM_TASK_ID, true>;
            multi = 1;
        }
    } else {
        if (p.n_steps > 1) return cudaErrorNotSupported;
    }
    int dev = 0;
    if (smem > 46 * 1024 && cudaGetDevice(&dev) == cudaSuccess && (dev >= 16 || smem > opted[multi][dev])) {
        // opt in above the 48 KB default (static tables aside), once per device
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (dev < 16) opted[multi][dev] = smem;
    }
    k<<<grid, block, smem, stream>>>(p);
    return cudaGetLastError();
}

template <class Real, int L, int MP, int MO>
static cudaError_t occ_V(int block, int smem, int* bps) {
    auto k = mrsim_dev::step_kernel<Real, L, MP, MO, MRSIM_TASK_ID>;
    if (smem > 46 * 1024) {  // opt in above the 48 KB default, leaving room for the static tables
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, block, smem);
}

// The instantiated (L, MP, MO) set; pick_variant (launch.h) maps configs onto it.
#define MRSIM_VARIANTS(X, MO)  \
    X(4, 2, MO) X(8, 2, MO) X(8, 4, MO) X(16, 3, MO) X(16, 8, MO)

template <class Real>
static cudaError_t launch_any(const mrsim_dev::StepParams<Real>& p, Variant v, int grid, int block, int smem,
                              cudaStream_t s) {
    if constexpr (MRSIM_TASK_ID != MRSIM_TASK_RWARE) {
        if (v.L == 1) {  // one thread per env (env_kernel.cuh)
            auto k = mrsim_dev::env_step_kernel<Real, MRSIM_TASK_ID>;
            if (smem + mrsim_dev::kEnvStaticSmem > 46 * 1024) {  // dynamic obs stage + static row/pose tables
                cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
            }
            k<<<grid, block, smem, s>>>(p);
            return cudaGetLastError();
        }
    }
#define MRSIM_CASE(l, mp, mo) \
    if (v.L == l && v.MP == mp && v.MO == mo) return launch_V<Real, l, mp, mo>(p, grid, block, smem, s);
    if constexpr (MRSIM_TASK_ID == MRSIM_TASK_RWARE) {
        MRSIM_VARIANTS(MRSIM_CASE, 6)
        MRSIM_VARIANTS(MRSIM_CASE, 16)
    } else {
        MRSIM_VARIANTS(MRSIM_CASE, 0)
    }
#undef MRSIM_CASE
    return cudaErrorInvalidValue;
}

template <class Real>
static cudaError_t occ_any(Variant v, int block, int smem, int* bps) {
    if constexpr (MRSIM_TASK_ID != MRSIM_TASK_RWARE) {
        if (v.L == 1) {
            auto k = mrsim_dev::env_step_kernel<Real, MRSIM_TASK_ID>;
            if (smem + mrsim_dev::kEnvStaticSmem > 46 * 1024) {
                cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                if (e != cudaSuccess) return e;
            }
            return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, block, smem);
        }
    }
#define MRSIM_CASE(l, mp, mo) \
    if (v.L == l && v.MP == mp && v.MO == mo) return occ_V<Real, l, mp, mo>(block, smem, bps);
    if constexpr (MRSIM_TASK_ID == MRSIM_TASK_RWARE) {
        MRSIM_VARIANTS(MRSIM_CASE, 6)
        MRSIM_VARIANTS(MRSIM_CASE, 16)
    } else {
        MRSIM_VARIANTS(MRSIM_CASE, 0)
    }
#undef MRSIM_CASE
    return cudaErrorInvalidValue;
}

template <>
cudaError_t launch_step<float, MRSIM_TASK_ID>(const mrsim_dev::StepParams<float>& p, Variant v, int grid, int block,
                                              int smem, cudaStream_t s) {
    return launch_any<float>(p, v, grid, block, smem, s);
}
template <>
cudaError_t launch_step<double, MRSIM_TASK_ID>(const mrsim_dev::StepParams<double>& p, Variant v, int grid,
                                               int block, int smem, cudaStream_t s) {
    return launch_any<double>(p, v, grid, block, smem, s);
}
template <>
cudaError_t step_occupancy<float, MRSIM_TASK_ID>(Variant v, int block, int smem, int* bps) {
    return occ_any<float>(v, block, smem, bps);
}
template <>
cudaError_t step_occupancy<double, MRSIM_TASK_ID>(Variant v, int block, int smem, int* bps) {
    return occ_any<double>(v, block, smem, bps);
}

template <>
cudaError_t launch_observe<float, MRSIM_TASK_ID>(const mrsim_cfg& c, const mrsim_dev::DevState<float>& s, float* obs,
                                                 long long B, int D, int bdim, int nf, int ni, cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>((B + 127) / 128);
    mrsim_dev::observe_kernel<float, MRSIM_TASK_ID><<<grid, 128, 0, st>>>(c, s, obs, B, c.num_robots, D, bdim, nf, ni);
    return cudaGetLastError();
}
template <>
cudaError_t launch_observe<double, MRSIM_TASK_ID>(const mrsim_cfg& c, const mrsim_dev::DevState<double>& s,
                                                  float* obs, long long B, int D, int bdim, int nf, int ni,
                                                  cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>((B + 127) / 128);
    mrsim_dev::observe_kernel<double, MRSIM_TASK_ID><<<grid, 128, 0, st>>>(c, s, obs, B, c.num_robots, D, bdim, nf, ni);
    return cudaGetLastError();
}

template <>
cudaError_t launch_reset<float, MRSIM_TASK_ID>(const mrsim_dev::ResetParams<float>& p, cudaStream_t s) {
    const int block = 128;
    const long long grid = (p.B + block - 1) / block;
    mrsim_dev::reset_kernel<float, MRSIM_TASK_ID><<<static_cast<unsigned>(grid), block, 0, s>>>(p);
    return cudaGetLastError();
}
template <>
cudaError_t launch_reset<double, MRSIM_TASK_ID>(const mrsim_dev::ResetParams<double>& p, cudaStream_t s) {
    const int block = 128;
    const long long grid = (p.B + block - 1) / block;
    mrsim_dev::reset_kernel<double, MRSIM_TASK_ID><<<static_cast<unsigned>(grid), block, 0, s>>>(p);
    return cudaGetLastError();
}

template <class Real>
static cudaError_t launch_policy_any(const mrsim_dev::PolicyParams<Real>& p, cudaStream_t s) {
    if (p.N <= mrsim_dev::kPolicyWarpMaxN) {  // one warp per env
        mrsim_dev::PolicyParams<Real> q = p;
        q.warp_bytes = mrsim_dev::policy_warp_bytes<Real>(p.N, p.maxw);
        int warps = mrsim_dev::kPolicyWarps;  // fewer warps per block when one env's buffers are large
        while (warps > 1 && warps * q.warp_bytes > 200 * 1024) warps >>= 1;
        const long long want = (p.B + warps - 1) / warps;
        const int smem = warps * q.warp_bytes;
        auto k = mrsim_dev::policy_warp_kernel<Real, MRSIM_TASK_ID>;
        if (smem > 48 * 1024) {
            const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
        }
        // grid-stride over envs: one full wave of resident blocks on this device
        int bps = 0;
        const cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, 32 * warps, smem);
        if (oe != cudaSuccess) return oe;
        const long long full = static_cast<long long>(p.num_sms) * (bps > 0 ? bps : 1);
        const unsigned grid = static_cast<unsigned>(want < full ? want : full);
        k<<<grid, 32 * warps, smem, s>>>(q);
        return cudaGetLastError();
    }
    mrsim_dev::PolicyParams<Real> q = p;
    q.tile_envs = mrsim_dev::policy_tile_envs<Real>(p.N, p.maxw);
    const int smem = mrsim_dev::policy_tile_bytes<Real>(q.tile_envs, p.N, p.maxw);
    const unsigned grid = static_cast<unsigned>((p.B + q.tile_envs - 1) / q.tile_envs);
    auto k = mrsim_dev::policy_tile_kernel<Real, MRSIM_TASK_ID>;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    k<<<grid, mrsim_dev::kPolicyTileThreads, smem, s>>>(q);
    return cudaGetLastError();
}
template <>
cudaError_t launch_policy<float, MRSIM_TASK_ID>(const mrsim_dev::PolicyParams<float>& p, cudaStream_t s) {
    return launch_policy_any<float>(p, s);
}
template <>
cudaError_t launch_policy<double, MRSIM_TASK_ID>(const mrsim_dev::PolicyParams<double>& p, cudaStream_t s) {
    return launch_policy_any<double>(p, s);
}

template <class Real>
static cudaError_t launch_scripted_any(const mrsim_dev::ScriptedParams<Real>& p, cudaStream_t s) {
    const long long want = (p.B + mrsim_dev::kPolicyWarps - 1) / mrsim_dev::kPolicyWarps;
    // grid cells as mrsim_set_policy_scripted sizes them (0.05 m, policy.hpp:253-255)
    const int cols = static_cast<int>((2.0 * p.c.arena_half_width) / 0.05);
    const int rows = static_cast<int>((2.0 * p.c.arena_half_height) / 0.05);
    mrsim_dev::ScriptedParams<Real> q = p;
    q.smem_stride = mrsim_dev::scripted_smem_stride(cols * rows);
    const int smem = q.smem_stride * mrsim_dev::kPolicyWarps;
    auto k = mrsim_dev::scripted_kernel<Real, MRSIM_TASK_ID>;
    if (smem > 48 * 1024) {
        const cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    // persistent: one full wave of resident blocks on this device (warps take envs from a counter)
    int bps = 0;
    cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k, 32 * mrsim_dev::kPolicyWarps, smem);
    if (oe != cudaSuccess) return oe;
    const long long full = static_cast<long long>(p.num_sms) * (bps > 0 ? bps : 1);
    const unsigned grid = static_cast<unsigned>(want < full ? want : full);
    k<<<grid, 32 * mrsim_dev::kPolicyWarps, smem, s>>>(q);
    return cudaGetLastError();
}
template <>
cudaError_t launch_scripted<float, MRSIM_TASK_ID>(const mrsim_dev::ScriptedParams<float>& p, cudaStream_t s) {
    return launch_scripted_any<float>(p, s);
}
template <>
cudaError_t launch_scripted<double, MRSIM_TASK_ID>(const mrsim_dev::ScriptedParams<double>& p, cudaStream_t s) {
    return launch_scripted_any<double>(p, s);
}

}  // namespace mrsim_host

#define MRSIM_DBG_CAT2(a, b) a##b
#define MRSIM_DBG_CAT(a, b) MRSIM_DBG_CAT2(a, b)
#ifdef MRSIM_QP_STATS  // diagnostic builds only: the QP counters of this task's kernels
extern "C" int MRSIM_DBG_CAT(mrsim_debug_qp_stats_task, MRSIM_TASK_ID)(unsigned long long* out8, int reset) {
    if (cudaMemcpyFromSymbol(out8, mrsim_dev::g_qp_stats, 64) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {0};
        cudaMemcpyToSymbol(mrsim_dev::g_qp_stats, z, 64);
    }
    return 0;
}
#endif

#ifdef MRSIM_TASK_STATS  // diagnostic builds only: the warp-task duration histogram of this task's kernels
extern "C" int MRSIM_DBG_CAT(mrsim_debug_task_hist_task, MRSIM_TASK_ID)(unsigned long long* out64, int reset) {
    if (cudaMemcpyFromSymbol(out64, mrsim_dev::g_task_hist, 512) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[64] = {0};
        cudaMemcpyToSymbol(mrsim_dev::g_task_hist, z, 512);
    }
    return 0;
}
extern "C" int MRSIM_DBG_CAT(mrsim_debug_warp_log_task, MRSIM_TASK_ID)(unsigned long long* out, int n_warps) {
    if (n_warps > mrsim_dev::kWarpLogMax) n_warps = mrsim_dev::kWarpLogMax;
    return cudaMemcpyFromSymbol(out, mrsim_dev::g_warp_log, 40 * n_warps) != cudaSuccess;
}
#endif
