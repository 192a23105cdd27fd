// launch.h — host-side launchers of the per-task kernel instantiations
// (one translation unit per task, compiled in parallel).
#pragma once

#include <cuda_runtime.h>

#include "policy.cuh"
#include "scripted.cuh"
#include "env_kernel.cuh"
#include "step_kernel.cuh"

namespace mrsim_host {

template <class Real>
inline void fill_consts(const mrsim_cfg& c, mrsim_dev::PhysConsts<Real>& k) {
    const double l = c.projection_distance;
    k.dt = Real(c.dt);
    k.v_max = Real(c.v_max);
    k.w_max = Real(c.omega_max);
    k.si_max = Real(c.si_max_speed);
    k.hw = Real(c.arena_half_width);
    k.hh = Real(c.arena_half_height);
    k.coll_r = Real(c.collision_radius);
    k.coll_r2 = Real(c.collision_radius * c.collision_radius);
    k.k_pos = Real(c.k_position);
    k.l = Real(l);
    k.inv_l = Real(1.0 / l);
    k.gamma = Real(c.barrier_gain);
    const double r_eff = c.safety_radius + 2.0 * l + c.discrete_margin;  // barrier.hpp:155
    k.r_eff2 = Real(r_eff * r_eff);
    const double m_eff = c.boundary_margin + l + c.discrete_margin;  // barrier.hpp:156
    k.wall_xmin = Real(-c.arena_half_width + m_eff);
    k.wall_xmax = Real(c.arena_half_width - m_eff);
    k.wall_ymin = Real(-c.arena_half_height + m_eff);
    k.wall_ymax = Real(c.arena_half_height - m_eff);
    const double ro = c.layout.rware_shelf_radius + l + c.discrete_margin;  // barrier.hpp:157
    k.obs_r_eff2 = Real(ro * ro);
    k.cap = Real(c.v_max + l * c.omega_max + 0.1);  // barrier.hpp:173
    k.tol = mrsim_dev::Prec<Real>::tol;
    k.k_rho = Real(c.k_rho);
    k.k_alpha = Real(c.k_alpha);
    k.k_beta = Real(c.k_beta);
    k.pose_ptol = Real(c.pose_position_tolerance);
    k.pose_htol = Real(c.pose_heading_tolerance);
}

// Kernel variant for a config: L lanes per env (lane per robot), MP pair-row
// slots per lane, MO obstacle-row slots per lane (rware only); L = 1 is the
// one-thread-per-env kernel (env_kernel.cuh) for teams of <= 4 robots without
// obstacle rows, on request (MRSIM_FLAG_ENV_PER_THREAD).
struct Variant {
    int L, MP, MO;
};
inline Variant pick_variant(const mrsim_cfg& c, unsigned flags = 0) {
    const int N = c.num_robots, P = N * (N - 1) / 2;
    Variant v;
    if (N <= mrsim_dev::kEnvNR && c.task != MRSIM_TASK_RWARE && (flags & MRSIM_FLAG_ENV_PER_THREAD)) {
        v.L = 1;
        v.MP = 0;
        v.MO = 0;
        return v;
    }
    v.L = N <= 4 ? 4 : (N <= 8 ? 8 : 16);
    const int need = (P + v.L - 1) / v.L;
    if (v.L == 4) v.MP = 2;
    else if (v.L == 8) v.MP = need <= 2 ? 2 : 4;
    else v.MP = need <= 3 ? 3 : 8;
    v.MO = c.task == MRSIM_TASK_RWARE ? (c.layout.rware_num_slots <= 6 ? 6 : 16) : 0;
    return v;
}

template <class Real, int TASK>
cudaError_t launch_step(const mrsim_dev::StepParams<Real>& p, Variant v, int grid, int block, int smem,
                        cudaStream_t stream);
template <class Real, int TASK>
cudaError_t step_occupancy(Variant v, int block, int smem, int* blocks_per_sm);
template <class Real, int TASK>
cudaError_t launch_observe(const mrsim_cfg& c, const mrsim_dev::DevState<Real>& s, float* obs, long long B, int D,
                           int bdim, int nf, int ni, cudaStream_t stream);
template <class Real, int TASK>
cudaError_t launch_reset(const mrsim_dev::ResetParams<Real>& p, cudaStream_t stream);
template <class Real, int TASK>
cudaError_t launch_policy(const mrsim_dev::PolicyParams<Real>& p, cudaStream_t stream);
template <class Real, int TASK>
cudaError_t launch_scripted(const mrsim_dev::ScriptedParams<Real>& p, cudaStream_t stream);

}  // namespace mrsim_host
