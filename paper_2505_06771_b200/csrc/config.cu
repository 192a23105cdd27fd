// config.cu — host-side ScenarioConfig for the C ABI: framework and task
// defaults, RunConfig-style overrides, layout keys and validation.
//
// Restates (paths relative to /root/reference/proj/include/mrsim):
//   SimParams defaults        core.hpp:79-99
//   ControllerGains defaults  controllers.hpp:13-31
//   BarrierConfig defaults    barrier.hpp:21-39
//   ScenarioConfig defaults   framework.hpp:129-166
//   Layout::defaults          layout.hpp:28-87
//   configure_defaults        scenarios/*.hpp
//   num_robots override       harness.hpp:82-89
//   validate                  framework.hpp:153-165, core.hpp:92-98, controllers.hpp:25-30,
//                             barrier.hpp:33-38, framework.hpp:34-57
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "mrsim_cuda.h"
#include "tasks.cuh"

namespace {

const char* kTaskNames[MRSIM_NUM_TASKS] = {"navigation", "predator_prey", "discovery", "rware",
                                           "foraging", "material_transport", "arctic_transport",
                                           "warehouse", "random_waypoints"};

void set4(double* d, double a, double b, double c, double e) {
    d[0] = a; d[1] = b; d[2] = c; d[3] = e;
}

void layout_defaults(mrsim_layout& y) {
    std::memset(&y, 0, sizeof y);
    y.spawn_margin = 0.25;
    y.spawn_separation_slack = 0.05;
    y.arctic_grid_cols = 8;
    y.arctic_grid_rows = 5;
    y.arctic_ground_cols_left = 1;
    y.arctic_ground_cols_right = 1;
    set4(y.arctic_goal_zone, 1.2, 1.6, -1.0, 1.0);
    set4(y.arctic_spawn_zone, -1.55, -1.25, -0.9, 0.9);
    y.arctic_normal_step = 0.2;
    y.arctic_fast_step = 0.3;
    y.arctic_slow_step = 0.1;
    y.discovery_num_landmarks = 6;
    y.discovery_landmark_margin = 0.3;
    y.discovery_sentinel[0] = -10.0;
    y.discovery_sentinel[1] = -10.0;
    y.foraging_num_resources = 2;
    y.foraging_radius = 0.3;
    y.foraging_resource_margin = 0.3;
    y.mt_circle_zone[0] = 0.2; y.mt_circle_zone[1] = 0.0; y.mt_circle_zone[2] = 0.3;
    set4(y.mt_rect_zone, 1.1, 1.55, -0.4, 0.4);
    set4(y.mt_dropoff_zone, -1.55, -1.05, -0.4, 0.4);
    y.mt_circle_mean = 75;
    y.mt_circle_variance = 10;
    y.mt_rect_mean = 15;
    y.mt_rect_variance = 4;
    y.navigation_goal_margin = 0.3;
    y.navigation_goal_separation = 0.4;
    y.navigation_on_goal_radius = 0.1;
    y.pp_tag_radius = 0.25;
    y.pp_prey_agility = 1.3;
    y.pp_prey_spawn_clearance = 0.35;
    y.pp_flash_steps = 2;
    const double slots[12] = {-0.2, -0.3, 0.25, -0.3, 0.7, -0.3, -0.2, 0.3, 0.25, 0.3, 0.7, 0.3};
    y.rware_num_slots = 6;
    for (int i = 0; i < 12; ++i) y.rware_slots[i] = slots[i];
    y.rware_slot_half = 0.12;
    y.rware_shelf_radius = 0.12;
    y.rware_num_shelves = 6;
    y.rware_request_size = 3;
    set4(y.rware_dropoff_zone, -1.55, -1.15, -0.4, 0.4);
    set4(y.warehouse_green_right, 1.15, 1.55, 0.15, 0.85);
    set4(y.warehouse_red_right, 1.15, 1.55, -0.85, -0.15);
    set4(y.warehouse_green_left, -1.55, -1.15, 0.15, 0.85);
    set4(y.warehouse_red_left, -1.55, -1.15, -0.85, -0.15);
    y.rwp_waypoint_margin = 0.2;
    y.rwp_arrival_tolerance = 0.05;
}

void set_coef(mrsim_cfg* c, int slot, double v) {
    c->coef[slot] = v;
    c->coef_present |= 1u << slot;
}

void set_het(mrsim_cfg* c, int kind, int mode, int rows, int cols, const double* vals) {
    c->het_kind = kind;
    c->het_obs_mode = mode;
    c->het_rows = rows;
    c->het_cols = cols;
    for (int i = 0; i < rows; ++i)
        for (int k = 0; k < cols; ++k) c->het[i][k] = vals[i * cols + k];
}

int fail(char* msg, int len, const std::string& text, int code) {
    if (msg && len > 0) {
        std::strncpy(msg, text.c_str(), static_cast<std::size_t>(len) - 1);
        msg[len - 1] = 0;
    }
    return code;
}

// Coefficients each task's transition reads via cfg.coefficient(name).
uint32_t required_coefs(int task) {
    const uint32_t v = 1u << MRSIM_COEF_VIOLATION;
    switch (task) {
        case MRSIM_TASK_NAVIGATION: return v | (1u << MRSIM_COEF_DIST);
        case MRSIM_TASK_PREDATOR_PREY: return v | (1u << MRSIM_COEF_TAG);
        case MRSIM_TASK_DISCOVERY: return v | (1u << MRSIM_COEF_SENSE) | (1u << MRSIM_COEF_TAG) | (1u << MRSIM_COEF_STEP);
        case MRSIM_TASK_RWARE: return v | (1u << MRSIM_COEF_DROPOFF);
        case MRSIM_TASK_FORAGING: return v | (1u << MRSIM_COEF_FORAGE);
        case MRSIM_TASK_MATERIAL_TRANSPORT:
            return v | (1u << MRSIM_COEF_LOAD) | (1u << MRSIM_COEF_DROPOFF) | (1u << MRSIM_COEF_STEP);
        case MRSIM_TASK_ARCTIC_TRANSPORT: return v | (1u << MRSIM_COEF_DIST) | (1u << MRSIM_COEF_STEP);
        case MRSIM_TASK_WAREHOUSE: return v | (1u << MRSIM_COEF_LOAD) | (1u << MRSIM_COEF_DELIVERY);
        default: return v;
    }
}

}  // namespace

namespace {
struct LayoutEnt {
    const char* key;
    double* d;
    int32_t* i;
    int arity;
};
// Layout keys (layout.hpp:28-87) -> fields of mrsim_layout; false if unknown.
bool layout_entry(mrsim_layout& y, const char* key, LayoutEnt* out) {
    const LayoutEnt table[] = {

        {"spawn.margin", &y.spawn_margin, nullptr, 1},
        {"spawn.separation_slack", &y.spawn_separation_slack, nullptr, 1},
        {"arctic.grid_cols", nullptr, &y.arctic_grid_cols, 1},
        {"arctic.grid_rows", nullptr, &y.arctic_grid_rows, 1},
        {"arctic.ground_cols_left", nullptr, &y.arctic_ground_cols_left, 1},
        {"arctic.ground_cols_right", nullptr, &y.arctic_ground_cols_right, 1},
        {"arctic.goal_zone", y.arctic_goal_zone, nullptr, 4},
        {"arctic.spawn_zone", y.arctic_spawn_zone, nullptr, 4},
        {"arctic.normal_step", &y.arctic_normal_step, nullptr, 1},
        {"arctic.fast_step", &y.arctic_fast_step, nullptr, 1},
        {"arctic.slow_step", &y.arctic_slow_step, nullptr, 1},
        {"discovery.num_landmarks", nullptr, &y.discovery_num_landmarks, 1},
        {"discovery.landmark_margin", &y.discovery_landmark_margin, nullptr, 1},
        {"discovery.sentinel", y.discovery_sentinel, nullptr, 2},
        {"foraging.num_resources", nullptr, &y.foraging_num_resources, 1},
        {"foraging.radius", &y.foraging_radius, nullptr, 1},
        {"foraging.resource_margin", &y.foraging_resource_margin, nullptr, 1},
        {"mt.circle_zone", y.mt_circle_zone, nullptr, 3},
        {"mt.rect_zone", y.mt_rect_zone, nullptr, 4},
        {"mt.dropoff_zone", y.mt_dropoff_zone, nullptr, 4},
        {"mt.circle_mean", &y.mt_circle_mean, nullptr, 1},
        {"mt.circle_variance", &y.mt_circle_variance, nullptr, 1},
        {"mt.rect_mean", &y.mt_rect_mean, nullptr, 1},
        {"mt.rect_variance", &y.mt_rect_variance, nullptr, 1},
        {"navigation.goal_margin", &y.navigation_goal_margin, nullptr, 1},
        {"navigation.goal_separation", &y.navigation_goal_separation, nullptr, 1},
        {"navigation.on_goal_radius", &y.navigation_on_goal_radius, nullptr, 1},
        {"pp.tag_radius", &y.pp_tag_radius, nullptr, 1},
        {"pp.prey_agility", &y.pp_prey_agility, nullptr, 1},
        {"pp.prey_spawn_clearance", &y.pp_prey_spawn_clearance, nullptr, 1},
        {"pp.flash_steps", nullptr, &y.pp_flash_steps, 1},
        {"rware.slot_half", &y.rware_slot_half, nullptr, 1},
        {"rware.shelf_radius", &y.rware_shelf_radius, nullptr, 1},
        {"rware.num_shelves", nullptr, &y.rware_num_shelves, 1},
        {"rware.request_size", nullptr, &y.rware_request_size, 1},
        {"rware.dropoff_zone", y.rware_dropoff_zone, nullptr, 4},
        {"warehouse.green_right", y.warehouse_green_right, nullptr, 4},
        {"warehouse.red_right", y.warehouse_red_right, nullptr, 4},
        {"warehouse.green_left", y.warehouse_green_left, nullptr, 4},
        {"warehouse.red_left", y.warehouse_red_left, nullptr, 4},
        {"rwp.waypoint_margin", &y.rwp_waypoint_margin, nullptr, 1},
        {"rwp.arrival_tolerance", &y.rwp_arrival_tolerance, nullptr, 1},
    };
    for (const LayoutEnt& e : table)
        if (std::strcmp(key, e.key) == 0) {
            *out = e;
            return true;
        }
    return false;
}
}  // namespace

extern "C" {

int mrsim_abi_version(void) { return MRSIM_ABI_VERSION; }

int mrsim_sizeof(int which) {
    switch (which) {
        case 0: return static_cast<int>(sizeof(mrsim_cfg));
        case 1: return static_cast<int>(sizeof(mrsim_layout));
        case 2: return static_cast<int>(sizeof(mrsim_env_state));
        case 3: return static_cast<int>(sizeof(mrsim_stats));
        case 4: return static_cast<int>(sizeof(mrsim_traj_record));
        default: return -1;
    }
}

const char* mrsim_task_name(int task) {
    return (task >= 0 && task < MRSIM_NUM_TASKS) ? kTaskNames[task] : "";
}

int mrsim_config_default(const char* scenario, mrsim_cfg* out) {
    if (!scenario || !out) return MRSIM_E_INVALID_ARGUMENT;
    int task = -1;
    for (int i = 0; i < MRSIM_NUM_TASKS; ++i)
        if (std::strcmp(scenario, kTaskNames[i]) == 0) task = i;
    if (task < 0) return MRSIM_E_INVALID_ARGUMENT;  // make_scenario: unknown scenario (scenario.hpp:218-227)
    mrsim_cfg& c = *out;
    std::memset(&c, 0, sizeof c);
    c.abi_version = MRSIM_ABI_VERSION;
    c.task = task;
    c.sub_steps = 10;
    c.controller = MRSIM_CONTROLLER_UNICYCLE_POSITION;
    c.barrier_enabled = 1;
    c.het_kind = MRSIM_HET_CLASS_ID;
    c.het_obs_mode = MRSIM_HET_OBS_NONE;
    c.action_noise_scale = 0.0;
    c.dt = 0.033; c.v_max = 0.2; c.omega_max = 3.6; c.si_max_speed = 0.15;
    c.arena_half_width = 1.6; c.arena_half_height = 1.0; c.collision_radius = 0.135;
    c.k_position = 1.0; c.projection_distance = 0.05; c.k_rho = 0.4; c.k_alpha = 1.5; c.k_beta = -0.3;
    c.pose_position_tolerance = 0.02; c.pose_heading_tolerance = 0.1;
    c.safety_radius = 0.17; c.barrier_gain = 100.0; c.boundary_margin = 0.05; c.discrete_margin = 0.002;
    layout_defaults(c.layout);
    auto steps = [&](int n, double s) {
        c.num_robots = n;
        for (int i = 0; i < n; ++i) c.step_sizes[i] = s;
    };
    switch (task) {
        case MRSIM_TASK_NAVIGATION:  // navigation.hpp:47-53
            steps(3, 0.2);
            c.max_steps = 100;
            set_coef(&c, MRSIM_COEF_DIST, -1.0);
            break;
        case MRSIM_TASK_PREDATOR_PREY:  // predator_prey.hpp:40-46
            steps(3, 0.2);
            c.max_steps = 100;
            set_coef(&c, MRSIM_COEF_TAG, 10.0);
            break;
        case MRSIM_TASK_DISCOVERY: {  // discovery.hpp:16-25
            steps(4, 0.2);
            c.max_steps = 100;
            const double v[] = {0.45, 0, 0.45, 0, 0, 0.25, 0, 0.25};
            set_het(&c, MRSIM_HET_CAPABILITY_SET, MRSIM_HET_OBS_FULL_TEAM, 4, 2, v);
            set_coef(&c, MRSIM_COEF_SENSE, 1.0);
            set_coef(&c, MRSIM_COEF_TAG, 5.0);
            set_coef(&c, MRSIM_COEF_STEP, -0.05);
            break;
        }
        case MRSIM_TASK_RWARE:  // rware.hpp:17-23
            steps(3, 0.2);
            c.max_steps = 100;
            set_coef(&c, MRSIM_COEF_DROPOFF, 1.0);
            break;
        case MRSIM_TASK_FORAGING: {  // foraging.hpp:15-25
            steps(3, 0.2);
            c.max_steps = 100;
            const double v[] = {1, 2, 3};
            set_het(&c, MRSIM_HET_CAPABILITY_SET, MRSIM_HET_OBS_FULL_TEAM, 3, 1, v);
            set_coef(&c, MRSIM_COEF_FORAGE, 1.0);
            break;
        }
        case MRSIM_TASK_MATERIAL_TRANSPORT: {  // material_transport.hpp:15-26
            c.num_robots = 4;
            c.max_steps = 70;
            const double v[] = {0.45, 5, 0.45, 5, 0.15, 15, 0.15, 15};
            set_het(&c, MRSIM_HET_CAPABILITY_SET, MRSIM_HET_OBS_FULL_TEAM, 4, 2, v);
            for (int i = 0; i < 4; ++i) c.step_sizes[i] = v[2 * i];
            set_coef(&c, MRSIM_COEF_LOAD, 0.25);
            set_coef(&c, MRSIM_COEF_DROPOFF, 0.75);
            set_coef(&c, MRSIM_COEF_STEP, -0.1);
            break;
        }
        case MRSIM_TASK_ARCTIC_TRANSPORT: {  // arctic_transport.hpp:116-125
            steps(4, c.layout.arctic_normal_step);
            c.max_steps = 100;
            const double v[] = {1, 0, 0, 1, 0, 0, 0, 1, 0, 0, 0, 1};
            set_het(&c, MRSIM_HET_CLASS_ID, MRSIM_HET_OBS_OWN, 4, 3, v);
            set_coef(&c, MRSIM_COEF_DIST, -0.05);
            set_coef(&c, MRSIM_COEF_STEP, -0.10);
            break;
        }
        case MRSIM_TASK_WAREHOUSE: {  // warehouse.hpp:14-23
            steps(4, 0.2);
            c.max_steps = 70;
            const double v[] = {1, 0, 1, 0, 0, 1, 0, 1};
            set_het(&c, MRSIM_HET_CLASS_ID, MRSIM_HET_OBS_OWN, 4, 2, v);
            set_coef(&c, MRSIM_COEF_LOAD, 1.0);
            set_coef(&c, MRSIM_COEF_DELIVERY, 3.0);
            break;
        }
        case MRSIM_TASK_RANDOM_WAYPOINTS:  // random_waypoints.hpp:15-21
            steps(4, 0.2);
            c.max_steps = 1000;
            break;
    }
    set_coef(&c, MRSIM_COEF_VIOLATION, 0.0);
    return MRSIM_OK;
}

int mrsim_config_set_num_robots(mrsim_cfg* c, int n, int tile_roster) {
    if (!c || n < 1) return MRSIM_E_INVALID_ARGUMENT;
    if (n > MRSIM_MAX_ROBOTS) return MRSIM_E_UNSUPPORTED;
    if (n == c->num_robots) return MRSIM_OK;
    if (c->het_rows > 0) {
        if (!tile_roster) return MRSIM_E_INVALID_ARGUMENT;  // fixed roster (harness.hpp:83-85)
        const int rows = c->het_rows;
        double het[MRSIM_MAX_ROBOTS][MRSIM_MAX_HET_COLS];
        double sizes[MRSIM_MAX_ROBOTS];
        std::memcpy(het, c->het, sizeof het);
        const int ns = c->num_robots;
        std::memcpy(sizes, c->step_sizes, sizeof sizes);
        for (int i = 0; i < n; ++i) {
            for (int k = 0; k < MRSIM_MAX_HET_COLS; ++k) c->het[i][k] = het[i % rows][k];
            c->step_sizes[i] = sizes[i % ns];
        }
        c->het_rows = n;
    } else {
        const double s0 = c->num_robots > 0 ? c->step_sizes[0] : 0.2;
        for (int i = 0; i < n; ++i) c->step_sizes[i] = s0;
    }
    for (int i = n; i < MRSIM_MAX_ROBOTS; ++i) c->step_sizes[i] = 0.0;
    c->num_robots = n;
    return MRSIM_OK;
}

int mrsim_config_set_layout(mrsim_cfg* c, const char* key, const double* v, int count) {
    if (!c || !key || (count > 0 && !v)) return MRSIM_E_INVALID_ARGUMENT;
    mrsim_layout& y = c->layout;
    if (std::strcmp(key, "rware.slots") == 0) {  // point list (layout.hpp:121-128)
        if (count % 2 != 0) return MRSIM_E_INVALID_ARGUMENT;
        if (count / 2 > MRSIM_MAX_SLOTS) return MRSIM_E_UNSUPPORTED;
        y.rware_num_slots = count / 2;
        for (int i = 0; i < 2 * MRSIM_MAX_SLOTS; ++i) y.rware_slots[i] = i < count ? v[i] : 0.0;
        return MRSIM_OK;
    }
    LayoutEnt e;
    if (!layout_entry(y, key, &e)) return MRSIM_E_INVALID_ARGUMENT;  // unknown key
    if (count != e.arity) return MRSIM_E_INVALID_ARGUMENT;
    for (int k = 0; k < count; ++k) {
        if (e.d) e.d[k] = v[k];
        else e.i[k] = static_cast<int32_t>(v[k]);  // Layout::integer (layout.hpp:105)
    }
    return MRSIM_OK;
}

int mrsim_config_get_layout(const mrsim_cfg* c, const char* key, double* out, int max_count) {
    if (!c || !key || !out) return -MRSIM_E_INVALID_ARGUMENT;
    mrsim_layout y = c->layout;
    if (std::strcmp(key, "rware.slots") == 0) {
        const int n = 2 * y.rware_num_slots;
        for (int k = 0; k < n && k < max_count; ++k) out[k] = y.rware_slots[k];
        return n;
    }
    LayoutEnt e;
    if (!layout_entry(y, key, &e)) return -MRSIM_E_INVALID_ARGUMENT;
    for (int k = 0; k < e.arity && k < max_count; ++k) out[k] = e.d ? e.d[k] : static_cast<double>(e.i[k]);
    return e.arity;
}

int mrsim_config_validate(const mrsim_cfg* cp, char* msg, int len) {
    if (!cp) return fail(msg, len, "null config", MRSIM_E_INVALID_ARGUMENT);
    const mrsim_cfg& c = *cp;
    const int IA = MRSIM_E_INVALID_ARGUMENT;
    if (c.abi_version != MRSIM_ABI_VERSION) return fail(msg, len, "mrsim_cfg: ABI version mismatch", IA);
    if (c.task < 0 || c.task >= MRSIM_NUM_TASKS) return fail(msg, len, "mrsim_cfg: unknown task", IA);
    if (c.num_robots < 1) return fail(msg, len, "ScenarioConfig: num_robots must be >= 1", IA);
    if (c.max_steps <= 0) return fail(msg, len, "ScenarioConfig: max_steps must be > 0", IA);
    if (c.sub_steps <= 0) return fail(msg, len, "ScenarioConfig: sub_steps must be > 0", IA);
    if (c.controller != MRSIM_CONTROLLER_UNICYCLE_POSITION && c.controller != MRSIM_CONTROLLER_UNICYCLE_POSE)
        return fail(msg, len, "ScenarioConfig: unknown controller", IA);
    if (c.action_noise_scale < 0) return fail(msg, len, "ScenarioConfig: action_noise_scale must be >= 0", IA);
    if (c.dt <= 0 || c.v_max <= 0 || c.omega_max <= 0 || c.si_max_speed <= 0 || c.arena_half_width <= 0 ||
        c.arena_half_height <= 0 || c.collision_radius <= 0)
        return fail(msg, len, "SimParams: all fields must be strictly positive", IA);
    if (c.collision_radius >= std::fmin(c.arena_half_width, c.arena_half_height))
        return fail(msg, len, "SimParams: collision_radius too large for arena", IA);
    if (c.k_position <= 0 || c.projection_distance <= 0)
        return fail(msg, len, "ControllerGains: k_position and projection_distance must be > 0", IA);
    if (!(c.k_rho > 0 && c.k_beta < 0 && c.k_alpha - c.k_rho > 0))
        return fail(msg, len, "ControllerGains: pose gains violate stability condition", IA);
    if (c.safety_radius < c.collision_radius)
        return fail(msg, len, "BarrierConfig: safety_radius < collision_radius", IA);
    if (c.barrier_gain <= 0) return fail(msg, len, "BarrierConfig: barrier_gain must be > 0", IA);
    if (!(c.het_obs_mode == MRSIM_HET_OBS_NONE && c.het_rows == 0)) {
        if (c.het_rows != c.num_robots) return fail(msg, len, "HeterogeneitySpec: row count != num_robots", IA);
        for (int i = 0; i < c.het_rows; ++i)
            for (int k = 0; k < c.het_cols; ++k)
                if (!std::isfinite(c.het[i][k])) return fail(msg, len, "HeterogeneitySpec: non-finite value", IA);
        if (c.het_kind == MRSIM_HET_CLASS_ID) {
            for (int i = 0; i < c.het_rows; ++i) {
                double sum = 0;
                for (int k = 0; k < c.het_cols; ++k) {
                    const double v = c.het[i][k];
                    if (v != 0.0 && v != 1.0)
                        return fail(msg, len, "HeterogeneitySpec: class rows must be one-hot", IA);
                    sum += v;
                }
                if (sum != 1.0) return fail(msg, len, "HeterogeneitySpec: class rows must be one-hot", IA);
            }
        }
    }
    const uint32_t need = required_coefs(c.task);
    if ((c.coef_present & need) != need)
        return fail(msg, len, std::string("ScenarioConfig: missing reward coefficient for scenario ") +
                                  mrsim_task_name(c.task), IA);
    // Task-specific preconditions the reference checks at use.
    const mrsim_layout& y = c.layout;
    const int US = MRSIM_E_UNSUPPORTED;
    if (c.task == MRSIM_TASK_RWARE && y.rware_num_slots < y.rware_num_shelves)
        return fail(msg, len, "rware: fewer slots than shelves in layout", IA);  // rware.hpp:30-31
    if ((c.task == MRSIM_TASK_DISCOVERY || c.task == MRSIM_TASK_FORAGING || c.task == MRSIM_TASK_MATERIAL_TRANSPORT ||
         c.task == MRSIM_TASK_ARCTIC_TRANSPORT || c.task == MRSIM_TASK_WAREHOUSE) &&
        c.het_rows != c.num_robots)
        return fail(msg, len, "scenario needs one heterogeneity row per robot", IA);
    if (c.task == MRSIM_TASK_ARCTIC_TRANSPORT && c.het_cols < 3)
        return fail(msg, len, "arctic_transport: heterogeneity rows must be one-hot over 3 classes", IA);
    if (c.task == MRSIM_TASK_MATERIAL_TRANSPORT && c.het_cols < 2)
        return fail(msg, len, "material_transport: heterogeneity rows need [step, capacity]", IA);
    if (c.task == MRSIM_TASK_WAREHOUSE && c.het_cols < 1) return fail(msg, len, "warehouse: empty roster", IA);
    if (c.task == MRSIM_TASK_DISCOVERY && c.het_cols < 2)
        return fail(msg, len, "discovery: heterogeneity rows need [sense, tag]", IA);
    // Device-path capacity.
    if (c.num_robots > MRSIM_MAX_ROBOTS) return fail(msg, len, "device path supports num_robots <= 16", US);
    if (c.het_cols > MRSIM_MAX_HET_COLS) return fail(msg, len, "device path supports <= 4 heterogeneity columns", US);
    if (y.discovery_num_landmarks < 0 || y.discovery_num_landmarks > MRSIM_MAX_LANDMARKS)
        return fail(msg, len, "discovery.num_landmarks out of device range", US);
    if (y.foraging_num_resources < 0 || y.foraging_num_resources > MRSIM_MAX_RESOURCES)
        return fail(msg, len, "foraging.num_resources out of device range", US);
    if (y.rware_num_slots > MRSIM_MAX_SLOTS || y.rware_num_shelves > 255 || y.rware_request_size > MRSIM_MAX_REQUESTS)
        return fail(msg, len, "rware layout out of device range", US);
    if (y.arctic_grid_cols < 1 || y.arctic_grid_rows < 1 || y.arctic_grid_cols * y.arctic_grid_rows > MRSIM_MAX_TILES)
        return fail(msg, len, "arctic grid out of device range", US);
    int nf = 0, ni = 0;
    mrsim_dev::task_fields(c, &nf, &ni);
    if (nf > mrsim_dev::kTfMax || ni > mrsim_dev::kTiMax) return fail(msg, len, "task state exceeds device staging", US);
    return MRSIM_OK;
}

int mrsim_obs_dim(const mrsim_cfg* c) { return c ? mrsim_dev::obs_dim_of(*c) : -1; }

int mrsim_task_fields(const mrsim_cfg* c, int* nf, int* ni) {
    if (!c || !nf || !ni) return MRSIM_E_INVALID_ARGUMENT;
    mrsim_dev::task_fields(*c, nf, ni);
    return MRSIM_OK;
}

}  // extern "C"
