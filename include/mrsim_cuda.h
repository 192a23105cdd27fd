/*
 * mrsim_cuda.h — C ABI of the B200-native batched Robotarium step.
 *
 * This is the drop-in boundary for the reference's batch engine
 * (/root/reference/proj/include/mrsim/batch.hpp). Every entry point below
 * names the reference interface it replaces (file:line, paths relative to
 * /root/reference/proj/include/mrsim). No C++ types, no exceptions and no
 * torch types cross this boundary: plain structs, pointers, sizes and
 * integer return codes (MRSIM_OK / MRSIM_E_*), with the message retrievable
 * through mrsim_last_error().
 *
 * Exception mapping (reference -> code):
 *   std::invalid_argument -> MRSIM_E_INVALID_ARGUMENT   (batch.hpp:226-237, framework.hpp:153-165)
 *   std::domain_error     -> MRSIM_E_DOMAIN             (barrier.hpp:73-74, core.hpp:103-104)
 *   std::runtime_error    -> MRSIM_E_RUNTIME            (scenario.hpp:113-115, spawn failures)
 *
 * Threading: one context per device, single driver thread per context
 * (the reference's WorkerPool has the same single-caller model,
 * batch.hpp:49-77). Calls taking a `stream` are stream-ordered and
 * asynchronous unless documented otherwise.
 */
#ifndef MRSIM_CUDA_H
#define MRSIM_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MRSIM_ABI_VERSION 2

/* ---- return codes ---- */
#define MRSIM_OK 0
#define MRSIM_E_INVALID_ARGUMENT 1
#define MRSIM_E_DOMAIN 2
#define MRSIM_E_RUNTIME 3
#define MRSIM_E_CUDA 4
#define MRSIM_E_UNSUPPORTED 5

/* ---- compile-time capacity of the device path ---- */
#define MRSIM_MAX_ROBOTS 16     /* 2N <= 32 QP variables: one warp per env at most */
#define MRSIM_MAX_LANDMARKS 16  /* discovery.num_landmarks */
#define MRSIM_MAX_RESOURCES 8   /* foraging.num_resources */
#define MRSIM_MAX_SLOTS 16      /* rware.slots / 2 */
#define MRSIM_MAX_REQUESTS 8    /* rware.request_size */
#define MRSIM_MAX_TILES 128     /* arctic.grid_cols * arctic.grid_rows */
#define MRSIM_MAX_HET_COLS 4

/* ---- tasks (scenarios/all.hpp:17-30) ---- */
#define MRSIM_TASK_NAVIGATION 0
#define MRSIM_TASK_PREDATOR_PREY 1
#define MRSIM_TASK_DISCOVERY 2
#define MRSIM_TASK_RWARE 3
#define MRSIM_TASK_FORAGING 4
#define MRSIM_TASK_MATERIAL_TRANSPORT 5
#define MRSIM_TASK_ARCTIC_TRANSPORT 6
#define MRSIM_TASK_WAREHOUSE 7
#define MRSIM_TASK_RANDOM_WAYPOINTS 8   /* throughput/determinism workload (random_waypoints.hpp) */
#define MRSIM_NUM_TASKS 9

/* ---- reward coefficient slots (ScenarioConfig::reward_coefficients, framework.hpp:139-151) ---- */
#define MRSIM_COEF_VIOLATION 0
#define MRSIM_COEF_DIST 1
#define MRSIM_COEF_TAG 2
#define MRSIM_COEF_SENSE 3
#define MRSIM_COEF_STEP 4
#define MRSIM_COEF_DROPOFF 5
#define MRSIM_COEF_FORAGE 6
#define MRSIM_COEF_LOAD 7
#define MRSIM_COEF_DELIVERY 8
#define MRSIM_NUM_COEF 9

/* HeterogeneitySpec enums (framework.hpp:21-22) */
#define MRSIM_HET_ROBOT_ID 0
#define MRSIM_HET_CLASS_ID 1
#define MRSIM_HET_CAPABILITY_SET 2
#define MRSIM_HET_OBS_NONE 0
#define MRSIM_HET_OBS_OWN 1
#define MRSIM_HET_OBS_FULL_TEAM 2

/* ControllerKind (framework.hpp:126): the projected-point position controller
 * (controllers.hpp:86-92, every benchmark scenario's default) or the polar
 * pose controller (controllers.hpp:68-82) with per-robot goal headings
 * (Scenario::waypoint_headings, scenario.hpp:168-177). */
#define MRSIM_CONTROLLER_UNICYCLE_POSITION 0
#define MRSIM_CONTROLLER_UNICYCLE_POSE 1

/* Flattened Layout table (layout.hpp:28-87). Keys map 1:1 to fields; integer
 * keys hold Layout::integer() = static_cast<int>(scalar) (layout.hpp:105). */
typedef struct mrsim_layout {
    double spawn_margin;              /* spawn.margin */
    double spawn_separation_slack;    /* spawn.separation_slack */
    int32_t arctic_grid_cols, arctic_grid_rows;
    int32_t arctic_ground_cols_left, arctic_ground_cols_right;
    double arctic_goal_zone[4];       /* xmin xmax ymin ymax */
    double arctic_spawn_zone[4];
    double arctic_normal_step, arctic_fast_step, arctic_slow_step;
    int32_t discovery_num_landmarks;
    int32_t foraging_num_resources;
    double discovery_landmark_margin;
    double discovery_sentinel[2];
    double foraging_radius, foraging_resource_margin;
    double mt_circle_zone[3];         /* cx cy radius */
    double mt_rect_zone[4];
    double mt_dropoff_zone[4];
    double mt_circle_mean, mt_circle_variance, mt_rect_mean, mt_rect_variance;
    double navigation_goal_margin, navigation_goal_separation, navigation_on_goal_radius;
    double pp_tag_radius, pp_prey_agility, pp_prey_spawn_clearance;
    int32_t pp_flash_steps;
    int32_t rware_num_slots;          /* rware.slots has 2*num_slots values */
    double rware_slots[2 * MRSIM_MAX_SLOTS];
    double rware_slot_half, rware_shelf_radius;
    int32_t rware_num_shelves, rware_request_size;
    double rware_dropoff_zone[4];
    double warehouse_green_right[4], warehouse_red_right[4];
    double warehouse_green_left[4], warehouse_red_left[4];
    double rwp_waypoint_margin, rwp_arrival_tolerance;
} mrsim_layout;

/* Flattened ScenarioConfig (framework.hpp:129-166) with SimParams
 * (core.hpp:79-99), ControllerGains (controllers.hpp:13-31) and BarrierConfig
 * (barrier.hpp:21-39; static obstacles are task-generated, rware only). */
typedef struct mrsim_cfg {
    int32_t abi_version;
    int32_t task;                   /* MRSIM_TASK_* */
    int32_t num_robots;
    int32_t max_steps;
    int32_t sub_steps;
    int32_t controller;             /* MRSIM_CONTROLLER_* */
    int32_t barrier_enabled;
    int32_t het_kind, het_obs_mode, het_rows, het_cols;
    int32_t _pad0;
    double action_noise_scale;
    double step_sizes[MRSIM_MAX_ROBOTS];
    double het[MRSIM_MAX_ROBOTS][MRSIM_MAX_HET_COLS];
    double coef[MRSIM_NUM_COEF];
    uint32_t coef_present;          /* bit c set <=> coefficient slot c is defined for the task */
    int32_t _pad1;
    /* SimParams */
    double dt, v_max, omega_max, si_max_speed, arena_half_width, arena_half_height, collision_radius;
    /* ControllerGains */
    double k_position, projection_distance, k_rho, k_alpha, k_beta;
    double pose_position_tolerance, pose_heading_tolerance;
    /* BarrierConfig */
    double safety_radius, barrier_gain, boundary_margin, discrete_margin;
    mrsim_layout layout;
} mrsim_cfg;

/* One environment, host side, in the reference's own precision (fp64):
 * EnvState (scenario.hpp:78-84) + Metrics (framework.hpp:111-117) + the
 * per-task state records (scenario.hpp:21-69). Used for parity (identical
 * initial states on both sides) and checkpoint/resume. */
typedef struct mrsim_env_state {
    int32_t num_robots;
    int32_t step_index;
    uint64_t rng_key;               /* EnvState::base_rng.key (ctr is always 0) */
    uint64_t seed;                  /* episode seed the env was reset from */
    int64_t episode;                /* episode index (harness seeds), -1 if reset from raw seeds */
    double x[MRSIM_MAX_ROBOTS], y[MRSIM_MAX_ROBOTS], theta[MRSIM_MAX_ROBOTS];
    /* Metrics */
    int64_t collisions;
    int64_t qp_infeasible;
    double scenario_metric;
    double min_pairwise_distance;
    int32_t success;
    int32_t _pad0;
    double episode_return;          /* sum of team rewards in the current episode */
    /* navigation */
    double goals[MRSIM_MAX_ROBOTS][2];
    /* predator_prey */
    double prey[2];
    int32_t flash_timer;
    /* discovery */
    int32_t num_landmarks;
    double landmarks[MRSIM_MAX_LANDMARKS][2];
    uint8_t sensed[MRSIM_MAX_LANDMARKS], tagged[MRSIM_MAX_LANDMARKS];
    /* rware */
    int32_t num_slots, num_requests;
    int32_t slot_shelf[MRSIM_MAX_SLOTS];
    int32_t carried[MRSIM_MAX_ROBOTS];
    int32_t requests[MRSIM_MAX_REQUESTS];
    /* foraging */
    int32_t num_resources;
    int32_t levels[MRSIM_MAX_RESOURCES];
    uint8_t foraged[MRSIM_MAX_RESOURCES];
    double resources[MRSIM_MAX_RESOURCES][2];
    /* material_transport */
    double circle_remaining, rect_remaining, delivered, total_initial;
    double loads[MRSIM_MAX_ROBOTS];
    /* arctic_transport */
    int32_t cols, rows;
    double goal_zone[4];
    int8_t tiles[MRSIM_MAX_TILES];
    /* warehouse */
    uint8_t loaded[MRSIM_MAX_ROBOTS];
    /* random_waypoints (RandomWaypointState, scenario.hpp:66-69) */
    double targets[MRSIM_MAX_ROBOTS][2];
    double target_headings[MRSIM_MAX_ROBOTS];
} mrsim_env_state;

/* Per-device partial episode statistics (EpisodeStats/RunSummary,
 * harness.hpp:157-194); combine across GPUs by summing and taking the min. */
typedef struct mrsim_stats {
    int64_t episodes;               /* completed episodes */
    int64_t env_steps;              /* env-steps taken since create */
    int64_t sum_collisions;
    int64_t sum_qp_infeasible;
    double sum_return, sum_return_sq;
    double sum_metric;
    double sum_success;
    double min_pairwise_distance;
} mrsim_stats;

typedef struct mrsim_ctx mrsim_ctx;

/* mrsim_create flags */
#define MRSIM_FLAG_FP64 1u          /* compute in fp64 (default: fp32) */
#define MRSIM_FLAG_AUTO_RESET 2u    /* reset done envs in-kernel (harness wave semantics) */
#define MRSIM_FLAG_ENV_PER_THREAD 4u /* teams of <= 4 robots without obstacle rows: step with one thread
                                       per env instead of the lane-per-robot kernel (same results; measured
                                       ~25% slower on B200: kept for A/B and tested) */

/* ---- configuration (host only, no device needed) ---- */

int mrsim_abi_version(void);
/* sizeof of the ABI structs (0 mrsim_cfg, 1 mrsim_layout, 2 mrsim_env_state,
 * 3 mrsim_stats, 4 mrsim_traj_record) so bindings can check their mirrors; -1 otherwise. */
int mrsim_sizeof(int which);
/* make_default_config(name) (scenario.hpp:230-236) incl. configure_defaults of the task. */
int mrsim_config_default(const char* scenario, mrsim_cfg* out);
/* RunConfig::num_robots override (harness.hpp:82-89). Fixed-roster tasks
 * refuse unless tile_roster != 0, in which case heterogeneity row i and step
 * size i become default row (i mod rows) (BASELINE.json configs 3-5). */
int mrsim_config_set_num_robots(mrsim_cfg* cfg, int num_robots, int tile_roster);
/* Layout::set (layout.hpp:130) for any key of the default table. */
int mrsim_config_set_layout(mrsim_cfg* cfg, const char* key, const double* values, int count);
/* Layout::get of a key (layout.hpp:98-105): writes up to max_count values,
 * returns the value count, or -MRSIM_E_INVALID_ARGUMENT for an unknown key. */
int mrsim_config_get_layout(const mrsim_cfg* cfg, const char* key, double* out, int max_count);
/* ScenarioConfig::validate (framework.hpp:153-165) plus device-path limits. */
int mrsim_config_validate(const mrsim_cfg* cfg, char* message, int message_len);
/* Per-robot observation length after het_augment (batch.hpp:143-151). */
int mrsim_obs_dim(const mrsim_cfg* cfg);
const char* mrsim_task_name(int task);
/* Per-env task-state words kept in HBM: nf compute-precision fields and ni
 * 32-bit integer words (used for the algorithmic-bytes roofline model). */
int mrsim_task_fields(const mrsim_cfg* cfg, int* nf, int* ni);

/* ---- batched environments on one device ---- */

int mrsim_create(const mrsim_cfg* cfg, int device, int64_t num_envs, uint32_t flags, mrsim_ctx** out);
void mrsim_destroy(mrsim_ctx* ctx);
const char* mrsim_last_error(const mrsim_ctx* ctx);
int64_t mrsim_num_envs(const mrsim_ctx* ctx);

/* reset_batch(cfg, seeds) (batch.hpp:240-259): env e <- reset_env(seeds[e])
 * (batch.hpp:153-160). seeds: host array of num_envs. obs_dev: device
 * [num_envs][N][D] fp32 or NULL. Synchronous (spawn failures are reported). */
int mrsim_reset_seeds(mrsim_ctx* ctx, const uint64_t* seeds, float* obs_dev, void* stream);
/* run_episodes wave seeding (harness.hpp:227-232): env e gets episode
 * first_episode + e, seed derive_episode_seed(root_seed, episode)
 * (harness.hpp:25-27). With MRSIM_FLAG_AUTO_RESET a done env continues with
 * episode += episode_stride. Synchronous. */
int mrsim_reset_episodes(mrsim_ctx* ctx, uint64_t root_seed, int64_t first_episode,
                         int64_t episode_stride, float* obs_dev, void* stream);

/* step_batch (batch.hpp:268-290) / step_env (batch.hpp:165-224) for every env.
 *   actions_dev : device int8 [num_envs][N] in 0..4, or NULL to let the
 *                 context's policy produce them on device: the harness random
 *                 policy policy_stream(seed_e, step, r).uniform_int(5)
 *                 (harness.hpp:29-34, policy.hpp:448-449) by default, or the
 *                 feedforward network set by mrsim_set_policy_feedforward
 *   obs_dev     : device fp32 [num_envs][N][D] (terminal obs on a done step, as
 *                 the reference returns), may be NULL
 *   reward_dev  : device fp32 [num_envs] team reward, may be NULL
 *   done_dev    : device uint8 [num_envs], may be NULL
 *   next_obs_dev: with MRSIM_FLAG_AUTO_RESET, the reset observation of done
 *                 envs (written only where done), may be NULL
 * Asynchronous on `stream`. A device-side error (invalid action, coincident
 * robots, spawn failure) is sticky: it is returned by the next synchronous
 * call (mrsim_sync) and later steps become no-ops. Each call flips the
 * context's state buffers and its warp-task counter (step serial & 1; a
 * scripted policy's planner kernel flips its own counter once per call too), so
 * a CUDA graph capturing mrsim_step must capture an even number of calls. */
int mrsim_step(mrsim_ctx* ctx, const int8_t* actions_dev, float* obs_dev, float* reward_dev,
               uint8_t* done_dev, float* next_obs_dev, void* stream);

/* A fused rollout: num_steps consecutive steps of every env in ONE launch, the actions drawn on
 * device by the harness random policy (policy_stream, harness.hpp:29-34) -- the same results,
 * bit for bit, as calling mrsim_step num_steps times with actions_dev = NULL (the on-device
 * equivalent of run_episodes' step loop, harness.hpp:255-286, without a host round trip between
 * steps). Each warp keeps its envs on chip across the steps, so the state crosses HBM once per
 * rollout and the launch's drain is paid once. Outputs are step-major, each may be NULL:
 *   obs_dev [num_steps][num_envs][N][D] fp32, reward_dev [num_steps][num_envs] fp32,
 *   done_dev [num_steps][num_envs] uint8.
 * Requires MRSIM_FLAG_FP64, the random policy (no feedforward / scripted policy), no trajectory
 * capture and the lane-group kernel (not MRSIM_FLAG_ENV_PER_THREAD): MRSIM_E_UNSUPPORTED otherwise.
 * Errors as mrsim_step (sticky, reported by mrsim_sync); a failing rollout is rolled back
 * as a whole, episode statistics included. */
int mrsim_rollout(mrsim_ctx* ctx, int num_steps, float* obs_dev, float* reward_dev, uint8_t* done_dev,
                  void* stream);
/* The same step with HOST buffers (the reference's std::vector<int> actions
 * and StepOutput fields): H2D of actions, step, D2H of obs/reward/done, sync.
 * Transactional: on error the batch state is left as before the call
 * (step_batch is pure, batch.hpp:267). Any output pointer may be NULL. */
int mrsim_step_host(mrsim_ctx* ctx, const int32_t* actions_host, float* obs_host,
                    double* reward_host, uint8_t* done_host, void* stream);
/* assemble_observations (batch.hpp:143-151) of the current state of every
 * env, on the device (obs_dev [num_envs][N][D] fp32, stream-ordered) or into
 * a host buffer (synchronous). */
int mrsim_observe(mrsim_ctx* ctx, float* obs_dev, void* stream);
int mrsim_observe_host(mrsim_ctx* ctx, float* obs_host);
/* Draw the harness random-policy actions for the current step into actions_dev. */
int mrsim_random_actions(mrsim_ctx* ctx, int8_t* actions_dev, void* stream);

/* ---- on-device policy (Policy / PolicySpec, policy.hpp:17-57, 445-486) ---- */
#define MRSIM_ACT_RELU 0      /* Activation (policy.hpp:60) */
#define MRSIM_ACT_TANH 1
#define MRSIM_ACT_IDENTITY 2
#define MRSIM_POLICY_MAX_LAYERS 8
#define MRSIM_POLICY_MAX_WIDTH 256
/* PolicyKind::FeedforwardFile with the weights already parsed
 * (FeedforwardWeights, policy.hpp:62-95; the text file format stays host
 * side): layer l maps dims[2l] -> dims[2l+1] inputs -> outputs with
 * activation[l]; `weights` holds, layer after layer, W (out x in, row-major,
 * as DenseLayer::w) then b (out). greedy != 0: argmax of the logits, else a
 * softmax sample from policy_stream (feedforward_sample:). Validates like
 * FeedforwardWeights::validate (chained dims, 5 logits) plus input dim ==
 * mrsim_obs_dim (forward's size check). Replaces the random policy used by
 * mrsim_step(actions_dev = NULL). Synchronous. */
int mrsim_set_policy_feedforward(mrsim_ctx* ctx, int num_layers, const int32_t* dims, const int32_t* activation,
                                 const double* weights, int greedy);
/* Back to PolicyKind::Random (the default). */
int mrsim_set_policy_random(mrsim_ctx* ctx);
/* The reference's scripted policies on device: PolicyKind::ScriptedGoal (grid
 * BFS planner toward Scenario::scripted_goal, policy.hpp:242-360) or
 * PolicyKind::PreyChaser (policy.hpp:362-416; predator_prey only, else
 * MRSIM_E_INVALID_ARGUMENT like resolve_scenario_config, harness.hpp:100-102). */
#define MRSIM_POLICY_SCRIPTED_GOAL 1
#define MRSIM_POLICY_PREY_CHASER 2
int mrsim_set_policy_scripted(mrsim_ctx* ctx, int kind);
/* The context policy's actions for the current step of every env (the
 * observation of the current state, i.e. the one the last reset/step
 * returned) into actions_dev [num_envs][N]. Asynchronous on `stream`. */
int mrsim_policy_actions(mrsim_ctx* ctx, int8_t* actions_dev, void* stream);
/* Wait for the context's work on `stream` and report sticky device errors. */
int mrsim_sync(mrsim_ctx* ctx, void* stream);

/* ---- on-device trajectory capture (run_episodes rows, harness.hpp:257-286;
 * TrajectoryRow, trajectory.hpp:38-82) ---- */
typedef struct mrsim_traj_record {
    double x, y, theta;             /* robot pose after the step */
    double reward;                  /* team reward of the step (StepOutput::team_reward) */
    double metric;                  /* Metrics::scenario_metric snapshot */
    int64_t collisions;             /* Metrics::collisions, cumulative within the episode */
    int32_t action;                 /* the action the robot took */
    int32_t done;                   /* StepOutput::done */
} mrsim_traj_record;
/* Start recording every subsequent mrsim_step (up to max_steps steps) into a
 * device buffer [max_steps][num_envs][N]; with actions_dev = NULL the policy's
 * actions are materialised so they can be recorded. Not allowed with
 * MRSIM_FLAG_AUTO_RESET (run_episodes waves do not auto-reset). Synchronous. */
int mrsim_capture_begin(mrsim_ctx* ctx, int64_t max_steps);
/* Steps recorded so far. */
int64_t mrsim_capture_steps(const mrsim_ctx* ctx);
/* Copy the records of envs [first_env, first_env+count) to host, laid out
 * [steps][count][N]. Synchronous. */
int mrsim_capture_read(mrsim_ctx* ctx, int64_t first_env, int64_t count, mrsim_traj_record* out);
/* Stop recording and free the buffer. */
int mrsim_capture_end(mrsim_ctx* ctx);
/* Host-side writer of the trajectory data section (write_trajectory,
 * trajectory.hpp:116-134): header_text (magic, config-hash, fields, column
 * line; built by the caller) verbatim, then one CSV row per (env, step,
 * robot), env-major, floats as %.17g. recs: [steps][envs][N]; rows carry env
 * index env_offset + e. append != 0 appends rows only (later waves). */
int mrsim_trajectory_write(const char* path, const char* header_text, const mrsim_traj_record* recs,
                           int64_t steps, int64_t envs, int num_robots, int64_t env_offset, int append);

/* Download / upload EnvState records of envs [first, first+count). Synchronous. */
int mrsim_get_env_states(mrsim_ctx* ctx, int64_t first, int64_t count, mrsim_env_state* out);
int mrsim_set_env_states(mrsim_ctx* ctx, int64_t first, int64_t count, const mrsim_env_state* in);
/* Per-device partial statistics over completed episodes. Synchronous. */
int mrsim_get_stats(mrsim_ctx* ctx, mrsim_stats* out);

/* ---- unit-level entry points (parity tests of the hot-path pieces) ---- */

/* solve_qp (qp.hpp:183-357) for `count` independent dense QPs of n <= 32
 * variables and m <= 64 rows: A [count][m][n], b [count][m], lo/hi/u_nom
 * [count][n] (|bound| >= 1e30 means unbounded). Outputs u [count][n],
 * status (0 optimal, 1 infeasible, 2 iteration limit), iterations. */
int mrsim_qp_solve_batch(int device, int fp64, int count, int n, int m, const double* A,
                         const double* b, const double* lo, const double* hi, const double* u_nom,
                         double tolerance, double* u_out, int32_t* status_out,
                         int32_t* iterations_out);
/* apply_barrier (barrier.hpp:132-205) for `count` teams of cfg->num_robots:
 * poses [count][N][3], nominal [count][N][2] (v, omega); optional static
 * obstacles [count][num_obstacles][3] (cx, cy, r) with masks
 * [count][num_obstacles]. Outputs commands [count][N][2], infeasible [count]. */
int mrsim_apply_barrier_batch(int device, int fp64, const mrsim_cfg* cfg, int count,
                              const double* poses, const double* nominal, int num_obstacles,
                              const double* obstacles, const uint64_t* obstacle_masks,
                              double* commands_out, int32_t* infeasible_out);

/* ---- measurement probe (roofline denominator) ---- */

/* Sustained FMA throughput of this device in FLOP/s (2 per FMA), fp64 or
 * fp32, from a register-resident FMA-chain kernel over all SMs. */
double mrsim_probe_fma_peak(int device, int fp64);

#ifdef __cplusplus
}
#endif

#endif /* MRSIM_CUDA_H */
