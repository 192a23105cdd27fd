/*
 * mrsim_oracle.h — TEST INFRASTRUCTURE (the checker, never the product).
 *
 * A plain-C, fp64, single-environment restatement of the reference's hot
 * path (/root/reference/proj/include/mrsim): SplitMix64 streams, the
 * position controller, build_barrier_constraints + fold_rows + solve_qp
 * (Goldfarb-Idnani with a re-factorised Gram matrix, exactly as qp.hpp),
 * apply_barrier, step_env and reset_env for the eight benchmark tasks, and
 * the observation layouts. Every function cites the reference file:line it
 * follows. Pinned bit-exactly against the reference itself
 * (oracle/_ref/libmrsim_ref.so) by tests/test_oracle.py, and against the
 * reference's own golden values (test_scenario_rules.cpp).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it. State and config use the C-ABI structs of include/mrsim_cuda.h.
 */
#ifndef MRSIM_ORACLE_H
#define MRSIM_ORACLE_H

#include <stdint.h>

#include "mrsim_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

uint64_t orc_mix64(uint64_t z);
uint64_t orc_key_from_seed(uint64_t seed);
uint64_t orc_fork(uint64_t key, uint64_t tag);
uint64_t orc_derive_episode_seed(uint64_t root, int episode);
int orc_policy_action(uint64_t episode_seed, int step, int robot);
/* count draws from SplitRng{fork(from_seed(seed), tag)}: kind 0 next_u64, 1 uniform, 2 normal, 3 uniform_int(n) */
void orc_rng_draws(uint64_t seed, uint64_t tag, int kind, uint64_t n, int count, double* out_f, uint64_t* out_u);

/* solve_qp (qp.hpp:183-357). A: m x n row-major. Returns 0 optimal, 1 infeasible, 2 iteration limit. */
int orc_solve_qp(int n, int m, const double* A, const double* b, const double* lo, const double* hi,
                 const double* u_nom, double tol, int max_iterations, double* u_out, int* iterations);

/* apply_barrier (barrier.hpp:132-205). poses [n][3], nominal [n][2], obstacles [nobs][3]. */
int orc_apply_barrier(const mrsim_cfg* cfg, int n, const double* poses, const double* nominal, int nobs,
                      const double* obstacles, const uint64_t* masks, double* commands, int* infeasible);

int orc_obs_dim(const mrsim_cfg* cfg);
/* reset_env (batch.hpp:153-160). Returns 0 or an MRSIM_E_* code with a message. */
int orc_reset_env(const mrsim_cfg* cfg, uint64_t seed, mrsim_env_state* out, char* err, int errlen);
/* step_env (batch.hpp:165-224) in place. obs: [N][D] or NULL. */
int orc_step_env(const mrsim_cfg* cfg, mrsim_env_state* st, const int32_t* actions, double* obs, double* reward,
                 int* done, char* err, int errlen);
/* assemble_observations (batch.hpp:143-151). */
int orc_observe(const mrsim_cfg* cfg, const mrsim_env_state* st, double* obs);
/* Policy::act for PolicyKind::FeedforwardFile (policy.hpp:445-480) on robot `robot`'s observation of
 * the current state; layers packed as in mrsim_set_policy_feedforward. */
int orc_policy_act(const mrsim_cfg* cfg, const mrsim_env_state* st, int robot, int num_layers, const int32_t* dims,
                   const int32_t* acts, const double* weights, int greedy);

#ifdef __cplusplus
}
#endif

#endif
