// oracle/ref_shim.cpp — TEST INFRASTRUCTURE, not product code.
//
// A thin extern "C" shim that compiles the UNMODIFIED reference headers
// (/root/reference/proj/include, header-only C++20, fp64) into
// oracle/_ref/libmrsim_ref.so so that the parity tests, smoke() and the
// bench's cpu_baseline / --impl reference leg can drive the reference itself
// from Python (ctypes). Nothing from the reference is copied: this file only
// #includes the reference headers from where they lie, through -I flags set
// by oracle/Makefile, with the reference's shipped flags
// (-O3 -DNDEBUG -std=gnu++20, no -march: CMakeLists.txt:1-19).
//
// The product path never links or loads this library.

#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "mrsim/harness.hpp"
#include "qp_oracle.hpp"
#include "mrsim_cuda.h"

using namespace mrsim;

namespace {

struct RefSpec {
    const char* scenario;
    int32_t num_robots;   // <= 0: task default
    int32_t tile_roster;  // tile fixed rosters row i <- row (i mod rows) (BASELINE configs 3-5)
    int32_t max_steps;    // <= 0: task default
    int32_t sub_steps;    // <= 0: default
    int32_t barrier;      // -1 default, 0 off, 1 on
    int32_t controller;   // -1 default, else MRSIM_CONTROLLER_*
    double noise;         // < 0: default
    const char* layout;   // "key v v v;key2 v ..." overrides, may be NULL
};

struct RefBatch {
    ScenarioConfig cfg;
    ScenarioPtr scenario;
    BatchWorldState state;
    std::vector<std::uint64_t> seeds;
    std::unique_ptr<WorkerPool> pool;
};

int code_of(const std::exception& e) {
    if (dynamic_cast<const std::invalid_argument*>(&e)) return MRSIM_E_INVALID_ARGUMENT;
    if (dynamic_cast<const std::domain_error*>(&e)) return MRSIM_E_DOMAIN;
    if (dynamic_cast<const std::runtime_error*>(&e)) return MRSIM_E_RUNTIME;
    return MRSIM_E_RUNTIME;
}

void put_err(char* err, int len, const std::exception& e) {
    if (err && len > 0) {
        std::strncpy(err, e.what(), static_cast<std::size_t>(len) - 1);
        err[len - 1] = 0;
    }
}

// Mirrors resolve_scenario_config (harness.hpp:71-103) with the BASELINE
// roster-tiling extension for fixed-roster tasks.
ScenarioConfig make_cfg(const RefSpec& s) {
    ScenarioConfig cfg = make_default_config(s.scenario);
    if (s.layout && *s.layout) {
        std::string text(s.layout);
        std::size_t pos = 0;
        while (pos < text.size()) {
            std::size_t end = text.find(';', pos);
            if (end == std::string::npos) end = text.size();
            std::istringstream is(text.substr(pos, end - pos));
            std::string key;
            is >> key;
            std::vector<double> vals;
            double v;
            while (is >> v) vals.push_back(v);
            if (!key.empty()) cfg.layout.set(key, vals);
            pos = end + 1;
        }
    }
    if (s.num_robots > 0 && s.num_robots != cfg.num_robots) {
        const int n = s.num_robots;
        if (!cfg.heterogeneity.values.empty()) {
            if (!s.tile_roster)
                throw std::invalid_argument("scenario '" + std::string(s.scenario) +
                                            "' has a fixed robot roster; num_robots cannot change");
            auto rows = cfg.heterogeneity.values;
            auto sizes = cfg.step_sizes;
            cfg.heterogeneity.values.clear();
            cfg.step_sizes.clear();
            for (int i = 0; i < n; ++i) {
                cfg.heterogeneity.values.push_back(rows[static_cast<std::size_t>(i) % rows.size()]);
                cfg.step_sizes.push_back(sizes[static_cast<std::size_t>(i) % sizes.size()]);
            }
        } else {
            cfg.step_sizes.assign(static_cast<std::size_t>(n),
                                  cfg.step_sizes.empty() ? 0.2 : cfg.step_sizes[0]);
        }
        cfg.num_robots = n;
    }
    if (s.max_steps > 0) cfg.max_steps = s.max_steps;
    if (s.sub_steps > 0) cfg.sub_steps = s.sub_steps;
    if (s.noise >= 0) cfg.action_noise_scale = s.noise;
    if (s.barrier >= 0) cfg.barrier_enabled = s.barrier != 0;
    if (s.controller >= 0)  // harness.hpp:95-96
        cfg.controller = s.controller == MRSIM_CONTROLLER_UNICYCLE_POSE ? ControllerKind::UnicyclePose
                                                                        : ControllerKind::UnicyclePosition;
    cfg.validate();
    return cfg;
}

int task_id(const std::string& name) {
    static const char* names[] = {"navigation", "predator_prey", "discovery", "rware",
                                  "foraging", "material_transport", "arctic_transport",
                                  "warehouse", "random_waypoints"};
    for (int i = 0; i < MRSIM_NUM_TASKS; ++i)
        if (name == names[i]) return i;
    return -1;
}

void copy4(double* dst, const Rect& r) {
    dst[0] = r.xmin; dst[1] = r.xmax; dst[2] = r.ymin; dst[3] = r.ymax;
}

void flatten(const ScenarioConfig& c, mrsim_cfg* o) {
    std::memset(o, 0, sizeof *o);
    o->abi_version = MRSIM_ABI_VERSION;
    o->task = task_id(c.scenario_name);
    o->num_robots = c.num_robots;
    o->max_steps = c.max_steps;
    o->sub_steps = c.sub_steps;
    o->controller = c.controller == ControllerKind::UnicyclePose ? MRSIM_CONTROLLER_UNICYCLE_POSE
                                                                : MRSIM_CONTROLLER_UNICYCLE_POSITION;
    o->barrier_enabled = c.barrier_enabled ? 1 : 0;
    o->het_kind = static_cast<int>(c.heterogeneity.kind);
    o->het_obs_mode = static_cast<int>(c.heterogeneity.obs_mode);
    o->het_rows = c.heterogeneity.rows();
    o->het_cols = c.heterogeneity.cols();
    o->action_noise_scale = c.action_noise_scale;
    for (int i = 0; i < c.num_robots && i < MRSIM_MAX_ROBOTS; ++i) o->step_sizes[i] = c.step_sizes[i];
    for (int i = 0; i < o->het_rows && i < MRSIM_MAX_ROBOTS; ++i)
        for (int k = 0; k < o->het_cols && k < MRSIM_MAX_HET_COLS; ++k)
            o->het[i][k] = c.heterogeneity.values[i][k];
    static const char* coef_names[MRSIM_NUM_COEF] = {"violation", "dist", "tag", "sense", "step",
                                                     "dropoff", "forage", "load", "delivery"};
    for (int k = 0; k < MRSIM_NUM_COEF; ++k) {
        auto it = c.reward_coefficients.find(coef_names[k]);
        if (it != c.reward_coefficients.end()) {
            o->coef[k] = it->second;
            o->coef_present |= 1u << k;
        }
    }
    const SimParams& p = c.params;
    o->dt = p.dt; o->v_max = p.v_max; o->omega_max = p.omega_max; o->si_max_speed = p.si_max_speed;
    o->arena_half_width = p.arena_half_width; o->arena_half_height = p.arena_half_height;
    o->collision_radius = p.collision_radius;
    const ControllerGains& g = c.gains;
    o->k_position = g.k_position; o->projection_distance = g.projection_distance;
    o->k_rho = g.k_rho; o->k_alpha = g.k_alpha; o->k_beta = g.k_beta;
    o->pose_position_tolerance = g.pose_position_tolerance;
    o->pose_heading_tolerance = g.pose_heading_tolerance;
    o->safety_radius = c.barrier.safety_radius; o->barrier_gain = c.barrier.barrier_gain;
    o->boundary_margin = c.barrier.boundary_margin; o->discrete_margin = c.barrier.discrete_margin;

    const Layout& L = c.layout;
    mrsim_layout& y = o->layout;
    y.spawn_margin = L.scalar("spawn.margin");
    y.spawn_separation_slack = L.scalar("spawn.separation_slack");
    y.arctic_grid_cols = L.integer("arctic.grid_cols");
    y.arctic_grid_rows = L.integer("arctic.grid_rows");
    y.arctic_ground_cols_left = L.integer("arctic.ground_cols_left");
    y.arctic_ground_cols_right = L.integer("arctic.ground_cols_right");
    copy4(y.arctic_goal_zone, L.rect("arctic.goal_zone"));
    copy4(y.arctic_spawn_zone, L.rect("arctic.spawn_zone"));
    y.arctic_normal_step = L.scalar("arctic.normal_step");
    y.arctic_fast_step = L.scalar("arctic.fast_step");
    y.arctic_slow_step = L.scalar("arctic.slow_step");
    y.discovery_num_landmarks = L.integer("discovery.num_landmarks");
    y.discovery_landmark_margin = L.scalar("discovery.landmark_margin");
    y.discovery_sentinel[0] = L.values("discovery.sentinel")[0];
    y.discovery_sentinel[1] = L.values("discovery.sentinel")[1];
    y.foraging_num_resources = L.integer("foraging.num_resources");
    y.foraging_radius = L.scalar("foraging.radius");
    y.foraging_resource_margin = L.scalar("foraging.resource_margin");
    Circle cz = L.circle("mt.circle_zone");
    y.mt_circle_zone[0] = cz.center.x; y.mt_circle_zone[1] = cz.center.y; y.mt_circle_zone[2] = cz.radius;
    copy4(y.mt_rect_zone, L.rect("mt.rect_zone"));
    copy4(y.mt_dropoff_zone, L.rect("mt.dropoff_zone"));
    y.mt_circle_mean = L.scalar("mt.circle_mean");
    y.mt_circle_variance = L.scalar("mt.circle_variance");
    y.mt_rect_mean = L.scalar("mt.rect_mean");
    y.mt_rect_variance = L.scalar("mt.rect_variance");
    y.navigation_goal_margin = L.scalar("navigation.goal_margin");
    y.navigation_goal_separation = L.scalar("navigation.goal_separation");
    y.navigation_on_goal_radius = L.scalar("navigation.on_goal_radius");
    y.pp_tag_radius = L.scalar("pp.tag_radius");
    y.pp_prey_agility = L.scalar("pp.prey_agility");
    y.pp_prey_spawn_clearance = L.scalar("pp.prey_spawn_clearance");
    y.pp_flash_steps = L.integer("pp.flash_steps");
    auto slots = L.points("rware.slots");
    y.rware_num_slots = static_cast<int32_t>(slots.size());
    for (std::size_t i = 0; i < slots.size() && i < MRSIM_MAX_SLOTS; ++i) {
        y.rware_slots[2 * i] = slots[i].x;
        y.rware_slots[2 * i + 1] = slots[i].y;
    }
    y.rware_slot_half = L.scalar("rware.slot_half");
    y.rware_shelf_radius = L.scalar("rware.shelf_radius");
    y.rware_num_shelves = L.integer("rware.num_shelves");
    y.rware_request_size = L.integer("rware.request_size");
    copy4(y.rware_dropoff_zone, L.rect("rware.dropoff_zone"));
    copy4(y.warehouse_green_right, L.rect("warehouse.green_right"));
    copy4(y.warehouse_red_right, L.rect("warehouse.red_right"));
    copy4(y.warehouse_green_left, L.rect("warehouse.green_left"));
    copy4(y.warehouse_red_left, L.rect("warehouse.red_left"));
    y.rwp_waypoint_margin = L.scalar("rwp.waypoint_margin");
    y.rwp_arrival_tolerance = L.scalar("rwp.arrival_tolerance");
}

void to_flat(const EnvState& s, std::uint64_t seed, mrsim_env_state* o) {
    std::memset(o, 0, sizeof *o);
    const int n = static_cast<int>(s.poses.size());
    o->num_robots = n;
    o->step_index = s.step_index;
    o->rng_key = s.base_rng.key;
    o->seed = seed;
    o->episode = -1;
    for (int i = 0; i < n && i < MRSIM_MAX_ROBOTS; ++i) {
        o->x[i] = s.poses[i].x;
        o->y[i] = s.poses[i].y;
        o->theta[i] = s.poses[i].theta;
    }
    o->collisions = s.metrics.collisions;
    o->qp_infeasible = s.metrics.qp_infeasible;
    o->scenario_metric = s.metrics.scenario_metric;
    o->min_pairwise_distance = s.metrics.min_pairwise_distance;
    o->success = s.metrics.success ? 1 : 0;
    std::visit(
        [&](const auto& st) {
            using T = std::decay_t<decltype(st)>;
            if constexpr (std::is_same_v<T, NavigationState>) {
                for (std::size_t i = 0; i < st.goals.size() && i < MRSIM_MAX_ROBOTS; ++i) {
                    o->goals[i][0] = st.goals[i].x;
                    o->goals[i][1] = st.goals[i].y;
                }
            } else if constexpr (std::is_same_v<T, PredatorPreyState>) {
                o->prey[0] = st.prey.x;
                o->prey[1] = st.prey.y;
                o->flash_timer = st.flash_timer;
            } else if constexpr (std::is_same_v<T, DiscoveryState>) {
                o->num_landmarks = static_cast<int32_t>(st.landmarks.size());
                for (std::size_t k = 0; k < st.landmarks.size() && k < MRSIM_MAX_LANDMARKS; ++k) {
                    o->landmarks[k][0] = st.landmarks[k].x;
                    o->landmarks[k][1] = st.landmarks[k].y;
                    o->sensed[k] = st.sensed[k] ? 1 : 0;
                    o->tagged[k] = st.tagged[k] ? 1 : 0;
                }
            } else if constexpr (std::is_same_v<T, RwareState>) {
                o->num_slots = static_cast<int32_t>(st.slot_shelf.size());
                o->num_requests = static_cast<int32_t>(st.requests.size());
                for (std::size_t k = 0; k < st.slot_shelf.size() && k < MRSIM_MAX_SLOTS; ++k)
                    o->slot_shelf[k] = st.slot_shelf[k];
                for (std::size_t k = 0; k < st.carried.size() && k < MRSIM_MAX_ROBOTS; ++k)
                    o->carried[k] = st.carried[k];
                for (std::size_t k = 0; k < st.requests.size() && k < MRSIM_MAX_REQUESTS; ++k)
                    o->requests[k] = st.requests[k];
            } else if constexpr (std::is_same_v<T, ForagingState>) {
                o->num_resources = static_cast<int32_t>(st.resources.size());
                for (std::size_t k = 0; k < st.resources.size() && k < MRSIM_MAX_RESOURCES; ++k) {
                    o->resources[k][0] = st.resources[k].x;
                    o->resources[k][1] = st.resources[k].y;
                    o->levels[k] = st.levels[k];
                    o->foraged[k] = st.foraged[k] ? 1 : 0;
                }
            } else if constexpr (std::is_same_v<T, MaterialTransportState>) {
                o->circle_remaining = st.circle_remaining;
                o->rect_remaining = st.rect_remaining;
                o->delivered = st.delivered;
                o->total_initial = st.total_initial;
                for (std::size_t k = 0; k < st.loads.size() && k < MRSIM_MAX_ROBOTS; ++k)
                    o->loads[k] = st.loads[k];
            } else if constexpr (std::is_same_v<T, ArcticState>) {
                o->cols = st.cols;
                o->rows = st.rows;
                copy4(o->goal_zone, st.goal_zone);
                for (std::size_t k = 0; k < st.tiles.size() && k < MRSIM_MAX_TILES; ++k)
                    o->tiles[k] = static_cast<int8_t>(st.tiles[k]);
            } else if constexpr (std::is_same_v<T, WarehouseState>) {
                for (std::size_t k = 0; k < st.loaded.size() && k < MRSIM_MAX_ROBOTS; ++k)
                    o->loaded[k] = st.loaded[k] ? 1 : 0;
            } else if constexpr (std::is_same_v<T, RandomWaypointState>) {
                for (std::size_t k = 0; k < st.targets.size() && k < MRSIM_MAX_ROBOTS; ++k) {
                    o->targets[k][0] = st.targets[k].x;
                    o->targets[k][1] = st.targets[k].y;
                    o->target_headings[k] = st.target_headings[k];
                }
            }
        },
        s.scenario);
}

void from_flat(const mrsim_env_state* o, const ScenarioConfig& cfg, EnvState& s) {
    const int n = o->num_robots;
    s.poses.assign(static_cast<std::size_t>(n), RobotPose{});
    for (int i = 0; i < n; ++i) s.poses[i] = {o->x[i], o->y[i], o->theta[i]};
    s.step_index = o->step_index;
    s.base_rng.key = o->rng_key;
    s.base_rng.ctr = 0;
    s.metrics.collisions = o->collisions;
    s.metrics.qp_infeasible = o->qp_infeasible;
    s.metrics.scenario_metric = o->scenario_metric;
    s.metrics.min_pairwise_distance = o->min_pairwise_distance;
    s.metrics.success = o->success != 0;
    switch (task_id(cfg.scenario_name)) {
        case MRSIM_TASK_NAVIGATION: {
            NavigationState st;
            for (int i = 0; i < n; ++i) st.goals.push_back({o->goals[i][0], o->goals[i][1]});
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_PREDATOR_PREY: {
            PredatorPreyState st;
            st.prey = {o->prey[0], o->prey[1]};
            st.flash_timer = o->flash_timer;
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_DISCOVERY: {
            DiscoveryState st;
            for (int k = 0; k < o->num_landmarks; ++k) {
                st.landmarks.push_back({o->landmarks[k][0], o->landmarks[k][1]});
                st.sensed.push_back(static_cast<char>(o->sensed[k]));
                st.tagged.push_back(static_cast<char>(o->tagged[k]));
            }
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_RWARE: {
            RwareState st;
            for (int k = 0; k < o->num_slots; ++k) st.slot_shelf.push_back(o->slot_shelf[k]);
            for (int k = 0; k < n; ++k) st.carried.push_back(o->carried[k]);
            for (int k = 0; k < o->num_requests; ++k) st.requests.push_back(o->requests[k]);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_FORAGING: {
            ForagingState st;
            for (int k = 0; k < o->num_resources; ++k) {
                st.resources.push_back({o->resources[k][0], o->resources[k][1]});
                st.levels.push_back(o->levels[k]);
                st.foraged.push_back(static_cast<char>(o->foraged[k]));
            }
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_MATERIAL_TRANSPORT: {
            MaterialTransportState st;
            st.circle_remaining = o->circle_remaining;
            st.rect_remaining = o->rect_remaining;
            st.delivered = o->delivered;
            st.total_initial = o->total_initial;
            for (int k = 0; k < n; ++k) st.loads.push_back(o->loads[k]);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_ARCTIC_TRANSPORT: {
            ArcticState st;
            st.cols = o->cols;
            st.rows = o->rows;
            st.goal_zone = {o->goal_zone[0], o->goal_zone[1], o->goal_zone[2], o->goal_zone[3]};
            for (int k = 0; k < o->cols * o->rows; ++k) st.tiles.push_back(o->tiles[k]);
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_WAREHOUSE: {
            WarehouseState st;
            for (int k = 0; k < n; ++k) st.loaded.push_back(static_cast<char>(o->loaded[k]));
            s.scenario = st;
            break;
        }
        case MRSIM_TASK_RANDOM_WAYPOINTS: {
            RandomWaypointState st;
            for (int k = 0; k < n; ++k) {
                st.targets.push_back({o->targets[k][0], o->targets[k][1]});
                st.target_headings.push_back(o->target_headings[k]);
            }
            s.scenario = st;
            break;
        }
        default:
            throw std::invalid_argument("ref_shim: unsupported scenario");
    }
}

void write_obs(const std::vector<std::vector<double>>& obs, double* out, int dim) {
    for (std::size_t r = 0; r < obs.size(); ++r)
        for (int k = 0; k < dim; ++k)
            out[r * static_cast<std::size_t>(dim) + static_cast<std::size_t>(k)] =
                k < static_cast<int>(obs[r].size()) ? obs[r][static_cast<std::size_t>(k)] : 0.0;
}

}  // namespace

extern "C" {

// ---- configuration ----

int ref_resolve_config(const RefSpec* spec, mrsim_cfg* out, char* err, int errlen) {
    try {
        flatten(make_cfg(*spec), out);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

void* ref_create(const RefSpec* spec, int workers, char* err, int errlen) {
    try {
        auto* b = new RefBatch;
        b->cfg = make_cfg(*spec);
        b->scenario = make_scenario(b->cfg.scenario_name);
        if (workers != 1) b->pool = std::make_unique<WorkerPool>(workers);
        return b;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return nullptr;
    }
}

void ref_destroy(void* h) { delete static_cast<RefBatch*>(h); }

int ref_flatten(void* h, mrsim_cfg* out) {
    flatten(static_cast<RefBatch*>(h)->cfg, out);
    return 0;
}

int ref_num_robots(void* h) { return static_cast<RefBatch*>(h)->cfg.num_robots; }

int ref_obs_dim(void* h) {
    auto* b = static_cast<RefBatch*>(h);
    EnvState st = reset_env(1, b->cfg, *b->scenario);
    return static_cast<int>(assemble_observations(st, b->cfg, *b->scenario)[0].size());
}

int ref_pool_size(void* h) {
    auto* b = static_cast<RefBatch*>(h);
    return b->pool ? b->pool->size() : 1;
}

// reset_batch (batch.hpp:240-259). obs_out: [B][N][D] or NULL.
int ref_reset(void* h, const std::uint64_t* seeds, int batch, double* obs_out, char* err, int errlen) {
    auto* b = static_cast<RefBatch*>(h);
    try {
        b->seeds.assign(seeds, seeds + batch);
        auto [state, out] = reset_batch(b->cfg, b->seeds, *b->scenario, b->pool.get());
        b->state = std::move(state);
        if (obs_out) {
            const int n = b->cfg.num_robots;
            const int d = static_cast<int>(out.obs[0][0].size());
            for (int e = 0; e < batch; ++e)
                write_obs(out.obs[e], obs_out + static_cast<std::size_t>(e) * n * d, d);
        }
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

// step_batch (batch.hpp:268-290). Outputs may be NULL. metrics_out (if not
// NULL): [B][6] = collisions, scenario_metric, success, min_pairwise, qp_infeasible, step_index.
int ref_step(void* h, const int32_t* actions, double* obs_out, double* reward_out,
             uint8_t* done_out, double* metrics_out, char* err, int errlen) {
    auto* b = static_cast<RefBatch*>(h);
    try {
        const int B = b->state.size();
        const int n = b->cfg.num_robots;
        std::vector<int> acts(actions, actions + static_cast<std::size_t>(B) * n);
        auto [next, outs] = step_batch(b->state, acts, b->cfg, *b->scenario, b->pool.get());
        b->state = std::move(next);
        for (int e = 0; e < B; ++e) {
            const StepOutput& o = outs[static_cast<std::size_t>(e)];
            if (obs_out) {
                const int d = static_cast<int>(o.obs[0].size());
                write_obs(o.obs, obs_out + static_cast<std::size_t>(e) * n * d, d);
            }
            if (reward_out) reward_out[e] = o.team_reward;
            if (done_out) done_out[e] = o.done ? 1 : 0;
            if (metrics_out) {
                double* m = metrics_out + static_cast<std::size_t>(e) * 6;
                m[0] = static_cast<double>(o.metrics.collisions);
                m[1] = o.metrics.scenario_metric;
                m[2] = o.metrics.success ? 1.0 : 0.0;
                m[3] = o.metrics.min_pairwise_distance;
                m[4] = static_cast<double>(o.metrics.qp_infeasible);
                m[5] = b->state.envs[static_cast<std::size_t>(e)].step_index;
            }
        }
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

int ref_batch_size(void* h) { return static_cast<RefBatch*>(h)->state.size(); }

int ref_get_states(void* h, int first, int count, mrsim_env_state* out) {
    auto* b = static_cast<RefBatch*>(h);
    for (int e = 0; e < count; ++e) {
        const std::size_t idx = static_cast<std::size_t>(first + e);
        to_flat(b->state.envs[idx], idx < b->seeds.size() ? b->seeds[idx] : 0, out + e);
    }
    return 0;
}

// Replace the batch with `count` envs from records (batch size becomes count).
int ref_set_states(void* h, int count, const mrsim_env_state* in, char* err, int errlen) {
    auto* b = static_cast<RefBatch*>(h);
    try {
        b->state.envs.assign(static_cast<std::size_t>(count), EnvState{});
        b->seeds.assign(static_cast<std::size_t>(count), 0);
        for (int e = 0; e < count; ++e) {
            from_flat(in + e, b->cfg, b->state.envs[static_cast<std::size_t>(e)]);
            b->seeds[static_cast<std::size_t>(e)] = in[e].seed;
        }
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

// Observations of the current state (assemble_observations, batch.hpp:143-151).
int ref_observe(void* h, double* obs_out) {
    auto* b = static_cast<RefBatch*>(h);
    const int n = b->cfg.num_robots;
    for (int e = 0; e < b->state.size(); ++e) {
        auto obs = assemble_observations(b->state.envs[static_cast<std::size_t>(e)], b->cfg, *b->scenario);
        const int d = static_cast<int>(obs[0].size());
        write_obs(obs, obs_out + static_cast<std::size_t>(e) * n * d, d);
    }
    return 0;
}

// Harness random policy for the current step of every env
// (harness.hpp:29-34 + policy.hpp:448-449), seeded by the env's reset seed.
int ref_random_actions(void* h, int32_t* out) {
    auto* b = static_cast<RefBatch*>(h);
    const int n = b->cfg.num_robots;
    for (int e = 0; e < b->state.size(); ++e) {
        const int step = b->state.envs[static_cast<std::size_t>(e)].step_index;
        for (int r = 0; r < n; ++r) {
            SplitRng prng = policy_stream(b->seeds[static_cast<std::size_t>(e)], step, r);
            out[static_cast<std::size_t>(e) * n + r] = static_cast<int32_t>(prng.uniform_int(kNumActions));
        }
    }
    return 0;
}

// Policy::act (policy.hpp:445-480) for every robot of every env on the
// current observation, seeded like run_episodes (harness.hpp:238-252).
// spec: a PolicySpec string ("random", "feedforward:<path>", ...).
int ref_policy_actions(void* h, const char* spec, int32_t* out, char* err, int errlen) {
    try {
        auto* b = static_cast<RefBatch*>(h);
        const int n = b->cfg.num_robots;
        Policy policy(PolicySpec::parse(spec));
        PolicyContext ctx;
        ctx.cfg = &b->cfg;
        ctx.scenario = b->scenario.get();
        for (int e = 0; e < b->state.size(); ++e) {
            const EnvState& env = b->state.envs[static_cast<std::size_t>(e)];
            const auto obs = assemble_observations(env, b->cfg, *b->scenario);
            ctx.state = &env;
            for (int r = 0; r < n; ++r) {
                ctx.robot = r;
                SplitRng prng = policy_stream(b->seeds[static_cast<std::size_t>(e)], env.step_index, r);
                out[static_cast<std::size_t>(e) * n + r] =
                    static_cast<int32_t>(policy.act(obs[static_cast<std::size_t>(r)], prng, ctx));
            }
        }
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

// CPU baseline: time `steps` step_batch calls (harness.hpp:356-362 style,
// steady_clock, setup excluded) with random-policy actions precomputed per step.
double ref_time_steps(void* h, int steps) {
    auto* b = static_cast<RefBatch*>(h);
    const int B = b->state.size();
    const int n = b->cfg.num_robots;
    std::vector<std::vector<int>> acts(static_cast<std::size_t>(steps),
                                       std::vector<int>(static_cast<std::size_t>(B) * n));
    for (int s = 0; s < steps; ++s)
        for (int e = 0; e < B; ++e) {
            const int step = b->state.envs[static_cast<std::size_t>(e)].step_index + s;
            for (int r = 0; r < n; ++r) {
                SplitRng prng = policy_stream(b->seeds[static_cast<std::size_t>(e)], step, r);
                acts[s][static_cast<std::size_t>(e) * n + r] = static_cast<int>(prng.uniform_int(kNumActions));
            }
        }
    auto t0 = std::chrono::steady_clock::now();
    for (int s = 0; s < steps; ++s) {
        auto [next, out] = step_batch(b->state, acts[static_cast<std::size_t>(s)], b->cfg, *b->scenario,
                                      b->pool.get());
        b->state = std::move(next);
    }
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
}

// ---- harness seeds / RNG ----

std::uint64_t ref_derive_episode_seed(std::uint64_t root, int episode) {
    return derive_episode_seed(root, episode);
}

int ref_policy_action(std::uint64_t seed, int step, int robot) {
    SplitRng prng = policy_stream(seed, step, robot);
    return static_cast<int>(prng.uniform_int(kNumActions));
}

// count draws of from_seed(seed).fork(tag) in each of the draw kinds
// kind 0 next_u64 (as double bits), 1 uniform, 2 normal, 3 uniform_int(n)
void ref_rng_draws(std::uint64_t seed, std::uint64_t tag, int kind, std::uint64_t n, int count,
                   double* out_f, std::uint64_t* out_u) {
    SplitRng r = SplitRng::from_seed(seed).fork(tag);
    for (int i = 0; i < count; ++i) {
        switch (kind) {
            case 0: out_u[i] = r.next_u64(); break;
            case 1: out_f[i] = r.uniform(); break;
            case 2: out_f[i] = r.normal(); break;
            default: out_u[i] = r.uniform_int(n); break;
        }
    }
}

// ---- unit pieces: QP and barrier ----

// solve_qp (qp.hpp:183-357). Returns status 0/1/2.
int ref_solve_qp(int n, int m, const double* A, const double* b, const double* lo, const double* hi,
                 const double* u_nom, double tol, int max_iter, double* u_out, int* iters,
                 double* kkt) {
    QuadraticProgram qp;
    qp.n = n;
    qp.u_nom.assign(u_nom, u_nom + n);
    qp.A.assign(A, A + static_cast<std::size_t>(m) * n);
    qp.b.assign(b, b + m);
    qp.lo.assign(lo, lo + n);
    qp.hi.assign(hi, hi + n);
    QpResult r = solve_qp(qp, tol, max_iter);
    for (int i = 0; i < n; ++i) u_out[i] = r.u[static_cast<std::size_t>(i)];
    if (iters) *iters = r.iterations;
    if (kkt) *kkt = r.kkt_residual;
    return r.status == QpStatus::Optimal ? 0 : (r.status == QpStatus::Infeasible ? 1 : 2);
}

// Brute-force active-set enumeration (tests/qp_oracle.hpp:54-115); returns 1 if found.
int ref_qp_enumeration(int n, int m, const double* A, const double* b, const double* u_nom,
                       double* u_out, double* objective) {
    QuadraticProgram qp;
    qp.n = n;
    qp.u_nom.assign(u_nom, u_nom + n);
    qp.A.assign(A, A + static_cast<std::size_t>(m) * n);
    qp.b.assign(b, b + m);
    qp.lo.assign(static_cast<std::size_t>(n), -kQpInf);
    qp.hi.assign(static_cast<std::size_t>(n), kQpInf);
    auto sol = testoracle::active_set_enumeration(qp);
    if (!sol) return 0;
    for (int i = 0; i < n; ++i) u_out[i] = sol->u[static_cast<std::size_t>(i)];
    *objective = sol->objective;
    return 1;
}

// The reference test generator random_feasible_qp (tests/qp_oracle.hpp:119-140),
// drawing `count` QPs in sequence from SplitRng::from_seed(seed). Rows padded
// to max_m x max_n.
void ref_random_qps(std::uint64_t seed, int count, int max_n, int max_m, int* n_out, int* m_out,
                    double* A_out, double* b_out, double* unom_out) {
    SplitRng rng = SplitRng::from_seed(seed);
    for (int t = 0; t < count; ++t) {
        QuadraticProgram qp = testoracle::random_feasible_qp(rng, max_n, max_m);
        n_out[t] = qp.n;
        m_out[t] = qp.rows();
        double* A = A_out + static_cast<std::size_t>(t) * max_m * max_n;
        for (int r = 0; r < qp.rows(); ++r)
            for (int i = 0; i < qp.n; ++i) A[r * max_n + i] = qp.A[static_cast<std::size_t>(r) * qp.n + i];
        for (int r = 0; r < qp.rows(); ++r) b_out[static_cast<std::size_t>(t) * max_m + r] = qp.b[r];
        for (int i = 0; i < qp.n; ++i) unom_out[static_cast<std::size_t>(t) * max_n + i] = qp.u_nom[i];
    }
}

// apply_barrier (barrier.hpp:132-205) with the handle's SimParams, gains and
// BarrierConfig (enabled flag from cfg.barrier_enabled).
int ref_apply_barrier(void* h, int n, const double* poses, const double* nominal, int num_obstacles,
                      const double* obstacles, const std::uint64_t* masks, double* cmds_out,
                      int* infeasible_out, double* kkt_out, char* err, int errlen) {
    auto* b = static_cast<RefBatch*>(h);
    try {
        std::vector<RobotPose> ps;
        std::vector<UnicycleVelocity> nom;
        for (int i = 0; i < n; ++i) {
            ps.push_back({poses[3 * i], poses[3 * i + 1], poses[3 * i + 2]});
            nom.push_back({nominal[2 * i], nominal[2 * i + 1]});
        }
        BarrierConfig bc = b->cfg.barrier;
        bc.enabled = b->cfg.barrier_enabled;
        for (int o = 0; o < num_obstacles; ++o) {
            bc.static_obstacles.push_back({{obstacles[3 * o], obstacles[3 * o + 1]}, obstacles[3 * o + 2]});
            bc.obstacle_masks.push_back(masks ? masks[o] : 0);
        }
        BarrierResult r = apply_barrier(ps, nom, bc, b->cfg.gains, b->cfg.params);
        for (int i = 0; i < n; ++i) {
            cmds_out[2 * i] = r.commands[static_cast<std::size_t>(i)].v;
            cmds_out[2 * i + 1] = r.commands[static_cast<std::size_t>(i)].omega;
        }
        *infeasible_out = r.infeasible ? 1 : 0;
        if (kkt_out) *kkt_out = r.kkt_residual;
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

// run_episodes (harness.hpp:216-300) writing the reference trajectory file
// (trajectory.hpp:116-134) for the given policy / controller / layout.
int ref_run_episodes_file(const char* scenario, std::uint64_t seed, int episodes, int batch, int num_robots,
                          int max_steps, const char* policy, const char* controller, const char* layout,
                          const char* out_path, char* err, int errlen) {
    try {
        RunConfig run;
        run.scenario = scenario;
        run.seed = seed;
        run.episodes = episodes;
        run.batch = batch;
        run.workers = 1;
        run.num_robots = num_robots;
        run.max_steps = max_steps;
        run.policy = policy;
        run.controller = controller ? controller : "";
        run.out = out_path;
        if (layout && *layout) {
            std::istringstream all(layout);
            std::string item;
            while (std::getline(all, item, ';')) {
                std::istringstream is(item);
                std::string key;
                is >> key;
                std::vector<double> vals;
                double v;
                while (is >> v) vals.push_back(v);
                if (!key.empty()) run.layout_overrides[key] = vals;
            }
        }
        run_episodes(run, true);
        return 0;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return code_of(e);
    }
}

// verify_trajectory (harness.hpp:444-518): 1 ok, 0 diverged (msg set).
int ref_verify_trajectory(const char* path, char* msg, int len, long long* first_row) {
    VerifyReport r = verify_trajectory(path);
    if (msg && len > 0) {
        std::strncpy(msg, r.message.c_str(), static_cast<std::size_t>(len) - 1);
        msg[len - 1] = 0;
    }
    if (first_row) *first_row = r.first_divergent_row;
    return r.ok ? 1 : 0;
}

// read_trajectory (trajectory.hpp:136-180): row count, or -code on a format error.
long ref_read_trajectory(const char* path, char* err, int errlen) {
    try {
        return static_cast<long>(read_trajectory(std::string(path)).rows.size());
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return -code_of(e);
    }
}

// run_episodes (harness.hpp:216-300) with the random policy, no file written.
// rows_out: [episodes*max_steps*N][11] = env, step, robot, x, y, theta, action,
// reward, done, collisions, metric. Returns the row count or -code.
long ref_run_episodes(const char* scenario, std::uint64_t seed, int episodes, int batch, int workers,
                      int num_robots, int max_steps, double* rows_out, long max_rows, char* err,
                      int errlen) {
    try {
        RunConfig run;
        run.scenario = scenario;
        run.seed = seed;
        run.episodes = episodes;
        run.batch = batch;
        run.workers = workers;
        run.num_robots = num_robots;
        run.max_steps = max_steps;
        RunSummary s = run_episodes(run, false);
        long k = 0;
        for (const auto& r : s.rows) {
            if (k >= max_rows) break;
            double* o = rows_out + k * 11;
            o[0] = r.env; o[1] = r.step; o[2] = r.robot; o[3] = r.x; o[4] = r.y; o[5] = r.theta;
            o[6] = r.action; o[7] = r.reward; o[8] = r.done ? 1 : 0;
            o[9] = static_cast<double>(r.collisions); o[10] = r.metric;
            ++k;
        }
        return k;
    } catch (const std::exception& e) {
        put_err(err, errlen, e);
        return -code_of(e);
    }
}

}  // extern "C"
