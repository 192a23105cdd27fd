// mrsim/cuda_batch.hpp — drop-in C++ host layer over the C ABI (mrsim_cuda.h)
// with the reference batch-engine shapes (batch.hpp:240-296):
//
//   auto [state, obs]  = mrsim::cuda::reset_batch(engine, cfg, seeds);
//   auto [next, outs]  = mrsim::cuda::step_batch(engine, state, actions, cfg);
//
// A caller of mrsim::reset_batch / mrsim::step_batch switches backends by
// calling mrsim::cuda::reset_batch / step_batch with the reference's own
// argument list (cfg, seeds, scenario, pool) / (state, actions, cfg, scenario,
// pool) -- one device context per (config, batch size) is created on first use
// and cached -- or by holding a mrsim::cuda::Engine explicitly. Types, value
// semantics (step_batch is pure) and exception types are the reference's; the
// caller's WorkerPool, when given, parallelises the host-side conversion of the
// reference's per-env objects (BatchWorldState, StepOutput) around the device step.
// Requires the reference headers on the include path (mrsim/batch.hpp) and
// linking libmrsim_cuda.so.
//
// For throughput the Engine also exposes the device-resident path
// (reset_episodes / step with device buffers) that skips the per-call state
// round trip the pure signature implies. mrsim::cuda::run_episodes(run) is the
// harness's run_episodes (harness.hpp:216-300) on the device, with the policy
// on device (mrsim::cuda::set_policy) and the rows recorded by the step; it
// returns the reference's RunSummary and writes the reference's trajectory file.
#pragma once

#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <variant>
#include <vector>

#include <algorithm>

#include "mrsim/batch.hpp"
#include "mrsim/harness.hpp"
#include "mrsim/policy.hpp"
#include "mrsim_cuda.h"

namespace mrsim::cuda {

namespace detail {

inline void throw_code(int code, const std::string& msg) {
    switch (code) {
        case MRSIM_OK: return;
        case MRSIM_E_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case MRSIM_E_DOMAIN: throw std::domain_error(msg);
        default: throw std::runtime_error(msg);
    }
}

inline int task_of(const std::string& name) {
    for (int t = 0; t < MRSIM_NUM_TASKS; ++t)
        if (name == mrsim_task_name(t)) return t;
    throw std::invalid_argument("mrsim::cuda: scenario '" + name + "' is not on the device path");
}

inline void rect4(double* d, const Rect& r) {
    d[0] = r.xmin; d[1] = r.xmax; d[2] = r.ymin; d[3] = r.ymax;
}

}  // namespace detail

/// Flatten a reference ScenarioConfig (framework.hpp:129-166) into the C ABI struct.
inline mrsim_cfg flatten(const ScenarioConfig& c) {
    mrsim_cfg o;
    std::memset(&o, 0, sizeof o);
    o.abi_version = MRSIM_ABI_VERSION;
    o.task = detail::task_of(c.scenario_name);
    o.num_robots = c.num_robots;
    o.max_steps = c.max_steps;
    o.sub_steps = c.sub_steps;
    o.controller = c.controller == ControllerKind::UnicyclePose ? MRSIM_CONTROLLER_UNICYCLE_POSE
                                                                : MRSIM_CONTROLLER_UNICYCLE_POSITION;
    o.barrier_enabled = c.barrier_enabled;
    o.het_kind = static_cast<int32_t>(c.heterogeneity.kind);
    o.het_obs_mode = static_cast<int32_t>(c.heterogeneity.obs_mode);
    o.het_rows = c.heterogeneity.rows();
    o.het_cols = c.heterogeneity.cols();
    if (c.num_robots > MRSIM_MAX_ROBOTS || o.het_cols > MRSIM_MAX_HET_COLS)
        throw std::invalid_argument("mrsim::cuda: config exceeds the device path capacity");
    o.action_noise_scale = c.action_noise_scale;
    for (int i = 0; i < c.num_robots; ++i) o.step_sizes[i] = c.step_sizes[static_cast<std::size_t>(i)];
    for (int i = 0; i < o.het_rows; ++i)
        for (int k = 0; k < o.het_cols; ++k) o.het[i][k] = c.heterogeneity.values[i][k];
    static const char* names[MRSIM_NUM_COEF] = {"violation", "dist", "tag", "sense", "step",
                                                "dropoff", "forage", "load", "delivery"};
    for (int k = 0; k < MRSIM_NUM_COEF; ++k) {
        auto it = c.reward_coefficients.find(names[k]);
        if (it != c.reward_coefficients.end()) {
            o.coef[k] = it->second;
            o.coef_present |= 1u << k;
        }
    }
    o.dt = c.params.dt; o.v_max = c.params.v_max; o.omega_max = c.params.omega_max;
    o.si_max_speed = c.params.si_max_speed; o.arena_half_width = c.params.arena_half_width;
    o.arena_half_height = c.params.arena_half_height; o.collision_radius = c.params.collision_radius;
    o.k_position = c.gains.k_position; o.projection_distance = c.gains.projection_distance;
    o.k_rho = c.gains.k_rho; o.k_alpha = c.gains.k_alpha; o.k_beta = c.gains.k_beta;
    o.pose_position_tolerance = c.gains.pose_position_tolerance;
    o.pose_heading_tolerance = c.gains.pose_heading_tolerance;
    o.safety_radius = c.barrier.safety_radius; o.barrier_gain = c.barrier.barrier_gain;
    o.boundary_margin = c.barrier.boundary_margin; o.discrete_margin = c.barrier.discrete_margin;
    const Layout& L = c.layout;
    mrsim_layout& y = o.layout;
    y.spawn_margin = L.scalar("spawn.margin");
    y.spawn_separation_slack = L.scalar("spawn.separation_slack");
    y.arctic_grid_cols = L.integer("arctic.grid_cols");
    y.arctic_grid_rows = L.integer("arctic.grid_rows");
    y.arctic_ground_cols_left = L.integer("arctic.ground_cols_left");
    y.arctic_ground_cols_right = L.integer("arctic.ground_cols_right");
    detail::rect4(y.arctic_goal_zone, L.rect("arctic.goal_zone"));
    detail::rect4(y.arctic_spawn_zone, L.rect("arctic.spawn_zone"));
    y.arctic_normal_step = L.scalar("arctic.normal_step");
    y.arctic_fast_step = L.scalar("arctic.fast_step");
    y.arctic_slow_step = L.scalar("arctic.slow_step");
    y.discovery_num_landmarks = L.integer("discovery.num_landmarks");
    y.discovery_landmark_margin = L.scalar("discovery.landmark_margin");
    y.discovery_sentinel[0] = L.values("discovery.sentinel").at(0);
    y.discovery_sentinel[1] = L.values("discovery.sentinel").at(1);
    y.foraging_num_resources = L.integer("foraging.num_resources");
    y.foraging_radius = L.scalar("foraging.radius");
    y.foraging_resource_margin = L.scalar("foraging.resource_margin");
    const Circle cz = L.circle("mt.circle_zone");
    y.mt_circle_zone[0] = cz.center.x; y.mt_circle_zone[1] = cz.center.y; y.mt_circle_zone[2] = cz.radius;
    detail::rect4(y.mt_rect_zone, L.rect("mt.rect_zone"));
    detail::rect4(y.mt_dropoff_zone, L.rect("mt.dropoff_zone"));
    y.mt_circle_mean = L.scalar("mt.circle_mean"); y.mt_circle_variance = L.scalar("mt.circle_variance");
    y.mt_rect_mean = L.scalar("mt.rect_mean"); y.mt_rect_variance = L.scalar("mt.rect_variance");
    y.navigation_goal_margin = L.scalar("navigation.goal_margin");
    y.navigation_goal_separation = L.scalar("navigation.goal_separation");
    y.navigation_on_goal_radius = L.scalar("navigation.on_goal_radius");
    y.pp_tag_radius = L.scalar("pp.tag_radius");
    y.pp_prey_agility = L.scalar("pp.prey_agility");
    y.pp_prey_spawn_clearance = L.scalar("pp.prey_spawn_clearance");
    y.pp_flash_steps = L.integer("pp.flash_steps");
    const auto slots = L.points("rware.slots");
    if (slots.size() > MRSIM_MAX_SLOTS) throw std::invalid_argument("mrsim::cuda: too many rware slots");
    y.rware_num_slots = static_cast<int32_t>(slots.size());
    for (std::size_t i = 0; i < slots.size(); ++i) {
        y.rware_slots[2 * i] = slots[i].x;
        y.rware_slots[2 * i + 1] = slots[i].y;
    }
    y.rware_slot_half = L.scalar("rware.slot_half");
    y.rware_shelf_radius = L.scalar("rware.shelf_radius");
    y.rware_num_shelves = L.integer("rware.num_shelves");
    y.rware_request_size = L.integer("rware.request_size");
    detail::rect4(y.rware_dropoff_zone, L.rect("rware.dropoff_zone"));
    detail::rect4(y.warehouse_green_right, L.rect("warehouse.green_right"));
    detail::rect4(y.warehouse_red_right, L.rect("warehouse.red_right"));
    detail::rect4(y.warehouse_green_left, L.rect("warehouse.green_left"));
    detail::rect4(y.warehouse_red_left, L.rect("warehouse.red_left"));
    y.rwp_waypoint_margin = L.scalar("rwp.waypoint_margin");
    y.rwp_arrival_tolerance = L.scalar("rwp.arrival_tolerance");
    return o;
}

/// EnvState (scenario.hpp:78-84) <-> mrsim_env_state.
/// Only the fields mrsim_set_env_states reads for the config's task are written
/// (no 2 KB clear per env).
inline void to_record(const EnvState& s, mrsim_env_state& o) {
    const int n = static_cast<int>(s.poses.size());
    o.num_robots = n;
    o.step_index = s.step_index;
    o.rng_key = s.base_rng.key;
    o.seed = 0;
    o.episode = -1;
    o.episode_return = 0.0;
    for (int i = 0; i < n; ++i) {
        o.x[i] = s.poses[i].x;
        o.y[i] = s.poses[i].y;
        o.theta[i] = s.poses[i].theta;
    }
    o.collisions = s.metrics.collisions;
    o.qp_infeasible = s.metrics.qp_infeasible;
    o.scenario_metric = s.metrics.scenario_metric;
    o.min_pairwise_distance = s.metrics.min_pairwise_distance;
    o.success = s.metrics.success;
    std::visit(
        [&](const auto& st) {
            using T = std::decay_t<decltype(st)>;
            if constexpr (std::is_same_v<T, NavigationState>) {
                for (std::size_t i = 0; i < st.goals.size(); ++i) {
                    o.goals[i][0] = st.goals[i].x;
                    o.goals[i][1] = st.goals[i].y;
                }
            } else if constexpr (std::is_same_v<T, PredatorPreyState>) {
                o.prey[0] = st.prey.x;
                o.prey[1] = st.prey.y;
                o.flash_timer = st.flash_timer;
            } else if constexpr (std::is_same_v<T, DiscoveryState>) {
                o.num_landmarks = static_cast<int32_t>(st.landmarks.size());
                for (std::size_t k = 0; k < st.landmarks.size(); ++k) {
                    o.landmarks[k][0] = st.landmarks[k].x;
                    o.landmarks[k][1] = st.landmarks[k].y;
                    o.sensed[k] = st.sensed[k] != 0;
                    o.tagged[k] = st.tagged[k] != 0;
                }
            } else if constexpr (std::is_same_v<T, RwareState>) {
                o.num_slots = static_cast<int32_t>(st.slot_shelf.size());
                o.num_requests = static_cast<int32_t>(st.requests.size());
                for (std::size_t k = 0; k < st.slot_shelf.size(); ++k) o.slot_shelf[k] = st.slot_shelf[k];
                for (std::size_t k = 0; k < st.carried.size(); ++k) o.carried[k] = st.carried[k];
                for (std::size_t k = 0; k < st.requests.size(); ++k) o.requests[k] = st.requests[k];
            } else if constexpr (std::is_same_v<T, ForagingState>) {
                o.num_resources = static_cast<int32_t>(st.resources.size());
                for (std::size_t k = 0; k < st.resources.size(); ++k) {
                    o.resources[k][0] = st.resources[k].x;
                    o.resources[k][1] = st.resources[k].y;
                    o.levels[k] = st.levels[k];
                    o.foraged[k] = st.foraged[k] != 0;
                }
            } else if constexpr (std::is_same_v<T, MaterialTransportState>) {
                o.circle_remaining = st.circle_remaining;
                o.rect_remaining = st.rect_remaining;
                o.delivered = st.delivered;
                o.total_initial = st.total_initial;
                for (std::size_t k = 0; k < st.loads.size(); ++k) o.loads[k] = st.loads[k];
            } else if constexpr (std::is_same_v<T, ArcticState>) {
                o.cols = st.cols;
                o.rows = st.rows;
                detail::rect4(o.goal_zone, st.goal_zone);
                for (std::size_t k = 0; k < st.tiles.size(); ++k) o.tiles[k] = static_cast<int8_t>(st.tiles[k]);
            } else if constexpr (std::is_same_v<T, WarehouseState>) {
                for (std::size_t k = 0; k < st.loaded.size(); ++k) o.loaded[k] = st.loaded[k] != 0;
            } else if constexpr (std::is_same_v<T, RandomWaypointState>) {
                for (std::size_t k = 0; k < st.targets.size(); ++k) {
                    o.targets[k][0] = st.targets[k].x;
                    o.targets[k][1] = st.targets[k].y;
                    o.target_headings[k] = st.target_headings[k];
                }
            }
        },
        s.scenario);
}
inline mrsim_env_state to_record(const EnvState& s) {
    mrsim_env_state o;
    std::memset(&o, 0, sizeof o);
    to_record(s, o);
    return o;
}

inline EnvState from_record(const mrsim_env_state& o, const ScenarioConfig& cfg) {
    EnvState s;
    const int n = o.num_robots;
    for (int i = 0; i < n; ++i) s.poses.push_back({o.x[i], o.y[i], o.theta[i]});
    s.step_index = o.step_index;
    s.base_rng.key = o.rng_key;
    s.metrics.collisions = o.collisions;
    s.metrics.qp_infeasible = o.qp_infeasible;
    s.metrics.scenario_metric = o.scenario_metric;
    s.metrics.min_pairwise_distance = o.min_pairwise_distance;
    s.metrics.success = o.success != 0;
    switch (detail::task_of(cfg.scenario_name)) {
        case MRSIM_TASK_NAVIGATION: {
            NavigationState st;
            for (int i = 0; i < n; ++i) st.goals.push_back({o.goals[i][0], o.goals[i][1]});
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_PREDATOR_PREY: {
            PredatorPreyState st;
            st.prey = {o.prey[0], o.prey[1]};
            st.flash_timer = o.flash_timer;
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_DISCOVERY: {
            DiscoveryState st;
            for (int k = 0; k < o.num_landmarks; ++k) {
                st.landmarks.push_back({o.landmarks[k][0], o.landmarks[k][1]});
                st.sensed.push_back(static_cast<char>(o.sensed[k]));
                st.tagged.push_back(static_cast<char>(o.tagged[k]));
            }
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_RWARE: {
            RwareState st;
            st.slot_shelf.assign(o.slot_shelf, o.slot_shelf + o.num_slots);
            st.carried.assign(o.carried, o.carried + n);
            st.requests.assign(o.requests, o.requests + o.num_requests);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_FORAGING: {
            ForagingState st;
            for (int k = 0; k < o.num_resources; ++k) {
                st.resources.push_back({o.resources[k][0], o.resources[k][1]});
                st.levels.push_back(o.levels[k]);
                st.foraged.push_back(static_cast<char>(o.foraged[k]));
            }
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_MATERIAL_TRANSPORT: {
            MaterialTransportState st;
            st.circle_remaining = o.circle_remaining;
            st.rect_remaining = o.rect_remaining;
            st.delivered = o.delivered;
            st.total_initial = o.total_initial;
            st.loads.assign(o.loads, o.loads + n);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_ARCTIC_TRANSPORT: {
            ArcticState st;
            st.cols = o.cols;
            st.rows = o.rows;
            st.goal_zone = {o.goal_zone[0], o.goal_zone[1], o.goal_zone[2], o.goal_zone[3]};
            st.tiles.assign(o.tiles, o.tiles + o.cols * o.rows);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_RANDOM_WAYPOINTS: {
            RandomWaypointState st;
            for (int i = 0; i < n; ++i) {
                st.targets.push_back({o.targets[i][0], o.targets[i][1]});
                st.target_headings.push_back(o.target_headings[i]);
            }
            s.scenario = st;
            break;
        }
        default: {
            WarehouseState st;
            st.loaded.assign(o.loaded, o.loaded + n);
            s.scenario = st;
            break;
        }
    }
    return s;
}

/// One device context. Owns the batch state in HBM.
class Engine {
public:
    Engine(const ScenarioConfig& cfg, int64_t num_envs, int device = 0, uint32_t flags = MRSIM_FLAG_FP64)
        : cfg_(flatten(cfg)), num_envs_(num_envs) {
        char msg[256] = {0};
        detail::throw_code(mrsim_config_validate(&cfg_, msg, sizeof msg), msg);
        detail::throw_code(mrsim_create(&cfg_, device, num_envs, flags, &ctx_), "mrsim_create failed");
    }
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;
    ~Engine() { mrsim_destroy(ctx_); }

    mrsim_ctx* ctx() const { return ctx_; }
    int64_t num_envs() const { return num_envs_; }
    int obs_dim() const { return mrsim_obs_dim(&cfg_); }
    void check(int code) const { detail::throw_code(code, mrsim_last_error(ctx_)); }

    std::vector<mrsim_env_state> download() const {
        std::vector<mrsim_env_state> rec(static_cast<std::size_t>(num_envs_));
        check(mrsim_get_env_states(ctx_, 0, num_envs_, rec.data()));
        return rec;
    }
    void download_into(std::vector<mrsim_env_state>& rec) const {
        rec.resize(static_cast<std::size_t>(num_envs_));
        check(mrsim_get_env_states(ctx_, 0, num_envs_, rec.data()));
    }
    void upload(const std::vector<mrsim_env_state>& rec) {
        check(mrsim_set_env_states(ctx_, 0, static_cast<int64_t>(rec.size()), rec.data()));
    }
    std::vector<mrsim_env_state>& scratch() { return scratch_; }  // reused per-env records

private:
    std::vector<mrsim_env_state> scratch_;
    mrsim_cfg cfg_;
    int64_t num_envs_;
    mrsim_ctx* ctx_ = nullptr;
};

namespace detail {
// fn(i) for i in [0, n): on the caller's WorkerPool in chunks when one is given.
template <class F>
inline void parallel_for(WorkerPool* pool, int64_t n, F&& fn) {
    if (!pool || pool->size() <= 1 || n < 2048) {
        for (int64_t i = 0; i < n; ++i) fn(i);
        return;
    }
    const int chunks = pool->size() * 4;
    const int64_t per = (n + chunks - 1) / chunks;
    pool->run(chunks, [&](int c) {
        const int64_t lo = c * per, hi = std::min<int64_t>(n, lo + per);
        for (int64_t i = lo; i < hi; ++i) fn(i);
    });
}
inline std::vector<std::vector<double>> unpack_obs(const float* o, int n, int d) {
    std::vector<std::vector<double>> out(static_cast<std::size_t>(n), std::vector<double>(static_cast<std::size_t>(d)));
    for (int r = 0; r < n; ++r)
        for (int k = 0; k < d; ++k) out[r][k] = o[r * d + k];
    return out;
}
}  // namespace detail

/// reset_batch (batch.hpp:240-259) on the device.
inline std::pair<BatchWorldState, ResetOutput> reset_batch(Engine& eng, const ScenarioConfig& cfg,
                                                           const std::vector<std::uint64_t>& seeds,
                                                           WorkerPool* pool = nullptr) {
    if (seeds.empty()) throw std::invalid_argument("reset_batch: seed list is empty");
    if (static_cast<int64_t>(seeds.size()) != eng.num_envs())
        throw std::invalid_argument("reset_batch: seed count != engine batch size");
    eng.check(mrsim_reset_seeds(eng.ctx(), seeds.data(), nullptr, nullptr));
    auto rec = eng.download();
    BatchWorldState state;
    ResetOutput out;
    const int n = cfg.num_robots, d = eng.obs_dim();
    std::vector<float> obs(static_cast<std::size_t>(eng.num_envs()) * n * d);
    eng.check(mrsim_observe_host(eng.ctx(), obs.data()));  // device-side assemble_observations
    state.envs.resize(rec.size());
    out.obs.resize(rec.size());
    detail::parallel_for(pool, eng.num_envs(), [&](int64_t e) {
        state.envs[static_cast<std::size_t>(e)] = from_record(rec[static_cast<std::size_t>(e)], cfg);
        out.obs[static_cast<std::size_t>(e)] = detail::unpack_obs(obs.data() + static_cast<std::size_t>(e) * n * d, n, d);
    });
    return {std::move(state), std::move(out)};
}

/// step_batch (batch.hpp:268-290) on the device: pure (input untouched), the
/// batch state is uploaded, stepped with the host actions and downloaded.
inline std::pair<BatchWorldState, std::vector<StepOutput>> step_batch(Engine& eng, const BatchWorldState& state,
                                                                      const std::vector<int>& actions,
                                                                      const ScenarioConfig& cfg,
                                                                      WorkerPool* pool = nullptr) {
    validate_actions(actions, state.size(), cfg.num_robots);  // reference message and ordering
    if (state.size() != eng.num_envs()) throw std::invalid_argument("step_batch: batch size != engine batch size");
    std::vector<mrsim_env_state>& rec = eng.scratch();
    rec.resize(state.envs.size());
    detail::parallel_for(pool, state.size(), [&](int64_t e) {
        to_record(state.envs[static_cast<std::size_t>(e)], rec[static_cast<std::size_t>(e)]);
    });
    eng.upload(rec);
    const int n = cfg.num_robots, d = eng.obs_dim();
    std::vector<float> obs(static_cast<std::size_t>(state.size()) * n * d);
    std::vector<double> rew(static_cast<std::size_t>(state.size()));
    std::vector<uint8_t> done(static_cast<std::size_t>(state.size()));
    std::vector<int32_t> acts(actions.begin(), actions.end());
    eng.check(mrsim_step_host(eng.ctx(), acts.data(), obs.data(), rew.data(), done.data(), nullptr));
    eng.download_into(rec);
    BatchWorldState next;
    next.envs.resize(state.envs.size());
    std::vector<StepOutput> outs(static_cast<std::size_t>(state.size()));
    detail::parallel_for(pool, state.size(), [&](int64_t e) {
        const std::size_t k = static_cast<std::size_t>(e);
        next.envs[k] = from_record(rec[k], cfg);
        StepOutput& o = outs[k];
        o.obs = detail::unpack_obs(obs.data() + k * n * d, n, d);
        o.team_reward = rew[k];
        o.done = done[k] != 0;
        o.metrics = next.envs[k].metrics;
    });
    return {std::move(next), std::move(outs)};
}

namespace detail {
// One device context per (flattened config, batch size, device), created on first use.
inline Engine& cached_engine(const ScenarioConfig& cfg, int64_t num_envs, int device = 0) {
    static std::mutex mu;
    static std::map<std::string, std::unique_ptr<Engine>> engines;
    const mrsim_cfg flat = flatten(cfg);  // zero-initialised, so the bytes are a key
    std::string key(reinterpret_cast<const char*>(&flat), sizeof flat);
    key += ":" + std::to_string(num_envs) + ":" + std::to_string(device);
    std::lock_guard<std::mutex> lk(mu);
    auto it = engines.find(key);
    if (it == engines.end()) it = engines.emplace(key, std::make_unique<Engine>(cfg, num_envs, device)).first;
    return *it->second;
}
}  // namespace detail

/// reset_batch with the reference's signature (batch.hpp:240-259): the device context for
/// (cfg, seeds.size()) is created on first use and cached. `scenario` is resolved on the
/// device from cfg.scenario_name (Scenario objects are stateless, scenario.hpp:132-134).
inline std::pair<BatchWorldState, ResetOutput> reset_batch(const ScenarioConfig& cfg,
                                                           const std::vector<std::uint64_t>& seeds,
                                                           const Scenario& scenario, WorkerPool* pool = nullptr) {
    (void)scenario;
    if (seeds.empty()) throw std::invalid_argument("reset_batch: seed list is empty");
    return reset_batch(detail::cached_engine(cfg, static_cast<int64_t>(seeds.size())), cfg, seeds, pool);
}

/// step_batch with the reference's signature (batch.hpp:268-290): pure, same exceptions.
inline std::pair<BatchWorldState, std::vector<StepOutput>> step_batch(const BatchWorldState& state,
                                                                      const std::vector<int>& actions,
                                                                      const ScenarioConfig& cfg,
                                                                      const Scenario& scenario,
                                                                      WorkerPool* pool = nullptr) {
    (void)scenario;
    validate_actions(actions, state.size(), cfg.num_robots);
    return step_batch(detail::cached_engine(cfg, state.size()), state, actions, cfg, pool);
}

/// The device policy used by steps without host actions (Policy / PolicySpec,
/// policy.hpp:17-57, 432-486): random (default), scripted_goal, prey_chaser, or
/// a feedforward network read by the reference's own FeedforwardWeights::load.
inline void set_policy(Engine& eng, const PolicySpec& spec) {
    switch (spec.kind) {
        case PolicyKind::Random: eng.check(mrsim_set_policy_random(eng.ctx())); return;
        case PolicyKind::ScriptedGoal: eng.check(mrsim_set_policy_scripted(eng.ctx(), MRSIM_POLICY_SCRIPTED_GOAL)); return;
        case PolicyKind::PreyChaser: eng.check(mrsim_set_policy_scripted(eng.ctx(), MRSIM_POLICY_PREY_CHASER)); return;
        case PolicyKind::FeedforwardFile: {
            const FeedforwardWeights w = FeedforwardWeights::load(spec.path);
            std::vector<int32_t> dims, acts;
            std::vector<double> flat;
            for (const DenseLayer& l : w.layers) {
                dims.push_back(l.in);
                dims.push_back(l.out);
                acts.push_back(l.activation == Activation::Relu ? MRSIM_ACT_RELU
                               : l.activation == Activation::Tanh ? MRSIM_ACT_TANH : MRSIM_ACT_IDENTITY);
                flat.insert(flat.end(), l.w.begin(), l.w.end());
                flat.insert(flat.end(), l.b.begin(), l.b.end());
            }
            eng.check(mrsim_set_policy_feedforward(eng.ctx(), static_cast<int>(w.layers.size()), dims.data(),
                                                   acts.data(), flat.data(), spec.greedy ? 1 : 0));
            return;
        }
    }
}

/// run_episodes (harness.hpp:216-300) on the device: waves of run.batch
/// episodes seeded derive_episode_seed(run.seed, episode), the policy producing
/// each step's actions on device, every (episode, step, robot) row recorded by
/// the step itself (mrsim_capture_*). Returns the reference's RunSummary (rows,
/// per-episode stats) and writes the reference's trajectory file with its own
/// build_header / write_trajectory.
inline RunSummary run_episodes(const RunConfig& run, bool write_file = true, int device = 0) {
    const ScenarioConfig cfg = resolve_scenario_config(run);
    const PolicySpec spec = PolicySpec::parse(run.policy);
    RunSummary summary;
    summary.scenario = run.scenario;
    summary.metric_name = scenario_metric_name(run.scenario);
    const int N = cfg.num_robots, T = cfg.max_steps;
    for (int wave_start = 0; wave_start < run.episodes; wave_start += run.batch) {
        const int wave = std::min(run.batch, run.episodes - wave_start);
        Engine eng(cfg, wave, device);
        set_policy(eng, spec);
        eng.check(mrsim_reset_episodes(eng.ctx(), run.seed, wave_start, wave, nullptr, nullptr));
        eng.check(mrsim_capture_begin(eng.ctx(), T));
        for (int t = 0; t < T; ++t) eng.check(mrsim_step(eng.ctx(), nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
        eng.check(mrsim_sync(eng.ctx(), nullptr));
        std::vector<mrsim_traj_record> rec(static_cast<std::size_t>(T) * wave * N);
        eng.check(mrsim_capture_read(eng.ctx(), 0, wave, rec.data()));
        const auto states = eng.download();
        for (int e = 0; e < wave; ++e) {
            double total = 0.0;
            for (int t = 0; t < T; ++t) {
                const mrsim_traj_record* at = rec.data() + (static_cast<std::size_t>(t) * wave + e) * N;
                total += at[0].reward;
                for (int r = 0; r < N; ++r) {
                    TrajectoryRow row;
                    row.env = wave_start + e;
                    row.step = t;
                    row.robot = r;
                    row.x = at[r].x;
                    row.y = at[r].y;
                    row.theta = at[r].theta;
                    row.action = at[r].action;
                    row.reward = at[r].reward;
                    row.done = at[r].done != 0;
                    row.collisions = at[r].collisions;
                    row.metric = at[r].metric;
                    summary.rows.push_back(row);
                }
            }
            const mrsim_env_state& s = states[static_cast<std::size_t>(e)];
            EpisodeStats st;
            st.total_reward = total;
            st.final_metric = s.scenario_metric;
            st.collisions = s.collisions;
            st.success = s.success != 0;
            st.min_pairwise_distance = s.min_pairwise_distance;
            st.qp_infeasible = s.qp_infeasible;
            summary.episodes.push_back(st);
        }
    }
    if (write_file) {
        summary.trajectory_path = run.out.empty() ? default_trajectory_path(run) : run.out;
        write_trajectory(summary.trajectory_path, build_header(run, cfg), summary.rows);
    }
    return summary;
}

}  // namespace mrsim::cuda
