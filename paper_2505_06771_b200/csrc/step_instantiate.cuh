// step_instantiate.cuh — included by step_<task>.cu with MRSIM_TASK_ID set:
// instantiates the fused step kernel for the three group widths and both
// precisions, and the reset kernel.
#pragma once

#include "launch.h"

namespace mrsim_host {

template <class Real, int L>
static cudaError_t launch_L(const mrsim_dev::StepParams<Real>& p, int grid, int block, int smem,
                            cudaStream_t stream) {
    auto k = mrsim_dev::step_kernel<Real, L, MRSIM_TASK_ID>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    k<<<grid, block, smem, stream>>>(p);
    return cudaGetLastError();
}

template <class Real, int L>
static cudaError_t occ_L(int block, int smem, int* bps) {
    auto k = mrsim_dev::step_kernel<Real, L, MRSIM_TASK_ID>;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps, k, block, smem);
}

template <>
cudaError_t launch_step<float, MRSIM_TASK_ID>(const mrsim_dev::StepParams<float>& p, int L, int grid, int block,
                                              int smem, cudaStream_t s) {
    if (L == 4) return launch_L<float, 4>(p, grid, block, smem, s);
    if (L == 8) return launch_L<float, 8>(p, grid, block, smem, s);
    return launch_L<float, 16>(p, grid, block, smem, s);
}
template <>
cudaError_t launch_step<double, MRSIM_TASK_ID>(const mrsim_dev::StepParams<double>& p, int L, int grid, int block,
                                               int smem, cudaStream_t s) {
    if (L == 4) return launch_L<double, 4>(p, grid, block, smem, s);
    if (L == 8) return launch_L<double, 8>(p, grid, block, smem, s);
    return launch_L<double, 16>(p, grid, block, smem, s);
}
template <>
cudaError_t step_occupancy<float, MRSIM_TASK_ID>(int L, int block, int smem, int* bps) {
    if (L == 4) return occ_L<float, 4>(block, smem, bps);
    if (L == 8) return occ_L<float, 8>(block, smem, bps);
    return occ_L<float, 16>(block, smem, bps);
}
template <>
cudaError_t step_occupancy<double, MRSIM_TASK_ID>(int L, int block, int smem, int* bps) {
    if (L == 4) return occ_L<double, 4>(block, smem, bps);
    if (L == 8) return occ_L<double, 8>(block, smem, bps);
    return occ_L<double, 16>(block, smem, bps);
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

}  // namespace mrsim_host
