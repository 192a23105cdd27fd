// tasks.cuh — the eight benchmark scenarios on the device: reset (fp64,
// bit-exact draw order), step sizes, static obstacles, transition, finalize
// and observation features. One set of functions per task, selected at
// compile time by the TASK template parameter of the step kernel. The ninth
// task, random_waypoints (random_waypoints.hpp), is the throughput workload
// of the paper's Table 1 / Fig. 3.
//
// Reference: scenarios/*.hpp, scenario.hpp:93-130 (sample_poses, spawn
// helpers), framework.hpp:61-76 (het_augment). Paths relative to
// /root/reference/proj/include/mrsim.
//
// State staging: during a step the group keeps one env's task state in
// shared memory as TF Real fields and TI 32-bit words, loaded from / stored
// to the SoA arrays tf[f][B], ti[w][B] in HBM. Per-task field maps:
//   navigation         TF: goals[2N]
//   predator_prey      TF: prey[2]                      TI: flash_timer
//   discovery          TF: landmarks[2K]                TI: sensed mask, tagged mask
//   rware              TI bytes: slot_shelf[S] | carried[N] | requests[R]
//   foraging           TF: resources[2M]                TI: foraged mask, levels[M]
//   material_transport TF: circle, rect, delivered, total_initial, loads[N]
//   arctic_transport   TI bytes: tiles[cols*rows]
//   warehouse          TI: loaded mask
//   random_waypoints   TF: targets[2N], target_headings[N]
#pragma once

#include <cmath>

#include "mrsim_device.cuh"

namespace mrsim_dev {

constexpr int kTfMax = 48;
constexpr int kTiMax = 32;

// Requests actually drawn at reset: min(request_size, num_shelves) (rware.hpp:38-42).
__host__ __device__ inline int rware_requests(const mrsim_layout& y) {
    const int r = y.rware_request_size < y.rware_num_shelves ? y.rware_request_size : y.rware_num_shelves;
    return r > 0 ? r : 0;
}

// Host+device field counts for a config.
__host__ __device__ inline void task_fields(const mrsim_cfg& c, int* nf, int* ni) {
    const int N = c.num_robots;
    const mrsim_layout& y = c.layout;
    *nf = 0;
    *ni = 0;
    switch (c.task) {
        case MRSIM_TASK_NAVIGATION: *nf = 2 * N; break;
        case MRSIM_TASK_PREDATOR_PREY: *nf = 2; *ni = 1; break;
        case MRSIM_TASK_DISCOVERY: *nf = 2 * y.discovery_num_landmarks; *ni = 2; break;
        case MRSIM_TASK_RWARE: *ni = (y.rware_num_slots + N + rware_requests(y) + 3) / 4; break;
        case MRSIM_TASK_FORAGING: *nf = 2 * y.foraging_num_resources; *ni = 1 + y.foraging_num_resources; break;
        case MRSIM_TASK_MATERIAL_TRANSPORT: *nf = 4 + N; break;
        case MRSIM_TASK_ARCTIC_TRANSPORT: *ni = (y.arctic_grid_cols * y.arctic_grid_rows + 3) / 4; break;
        case MRSIM_TASK_WAREHOUSE: *ni = 1; break;
        case MRSIM_TASK_RANDOM_WAYPOINTS: *nf = 3 * N; break;
        default: break;
    }
}

// byte view of the TI words (little-endian packing)
__device__ __forceinline__ int ti_byte(const int* ti, int b) { return (ti[b >> 2] >> (8 * (b & 3))) & 0xff; }
__device__ __forceinline__ void ti_set_byte(int* ti, int b, int v) {
    const int sh = 8 * (b & 3);
    ti[b >> 2] = (ti[b >> 2] & ~(0xff << sh)) | ((v & 0xff) << sh);
}

// Rect helpers on layout quadruples (core.hpp:32-45).
template <class Real>
__device__ __forceinline__ bool rect_contains(const double* r, Real x, Real y) {
    return x >= Real(r[0]) && x <= Real(r[1]) && y >= Real(r[2]) && y <= Real(r[3]);
}

// ---------------------------------------------------------------------------
// Reset (fp64, one lane). Mirrors Scenario::reset of each task plus
// sample_poses (scenario.hpp:95-118). Writes poses and task staging.
// Returns 0 or a DevErr code (with *bad_robot set for spawn failures).
// ---------------------------------------------------------------------------
struct ResetOut {
    double x[MRSIM_MAX_ROBOTS], y[MRSIM_MAX_ROBOTS], th[MRSIM_MAX_ROBOTS];
    double tf[kTfMax];
    int ti[kTiMax];
};

__device__ inline int sample_poses_dev(int n, double xmin, double xmax, double ymin, double ymax, double min_sep,
                                       Rng& rng, ResetOut& o, int* bad) {
    for (int i = 0; i < n; ++i) {
        bool placed = false;
        for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
            const double px = rng.uniform(xmin, xmax);
            const double py = rng.uniform(ymin, ymax);
            const double pt = __dmul_rn(3.14159265358979323846, __dsub_rn(1.0, __dmul_rn(2.0, rng.uniform())));
            bool ok = true;
            for (int q = 0; q < i; ++q)
                if (hypot(px - o.x[q], py - o.y[q]) < min_sep) { ok = false; break; }
            if (ok) {
                o.x[i] = px;
                o.y[i] = py;
                o.th[i] = pt;
                placed = true;
            }
        }
        if (!placed) {
            *bad = i;
            return kErrSpawn;
        }
    }
    return 0;
}

// RandomWaypointsScenario::draw_target + a heading (random_waypoints.hpp:24-27, 34-35, 62-63)
__device__ __forceinline__ void rwp_draw(const mrsim_cfg& c, Rng& rng, double& tx, double& ty, double& th) {
    const double m = c.layout.rwp_waypoint_margin;
    const double hw = c.arena_half_width, hh = c.arena_half_height;
    tx = rng.uniform(-hw + m, hw - m);
    ty = rng.uniform(-hh + m, hh - m);
    th = __dmul_rn(3.14159265358979323846, __dsub_rn(1.0, __dmul_rn(2.0, rng.uniform())));
}

template <int TASK>
__device__ inline int reset_task(const mrsim_cfg& c, uint64_t key, ResetOut& o, int* bad) {
    Rng rng{fork_key(key, 0), 0};  // reset_stream = base_rng.fork(0) (scenario.hpp:87-88)
    const mrsim_layout& y = c.layout;
    const int N = c.num_robots;
    const double hw = c.arena_half_width, hh = c.arena_half_height;
    const double sm = y.spawn_margin;
    const double sep = c.safety_radius + y.spawn_separation_slack;  // scenario.hpp:124-126
    for (int w = 0; w < kTiMax; ++w) o.ti[w] = 0;
    int err;
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {
        err = sample_poses_dev(N, y.arctic_spawn_zone[0], y.arctic_spawn_zone[1], y.arctic_spawn_zone[2],
                               y.arctic_spawn_zone[3], sep, rng, o, bad);
    } else {
        err = sample_poses_dev(N, -hw + sm, hw - sm, -hh + sm, hh - sm, sep, rng, o, bad);
    }
    if (err) return err;
    if (TASK == MRSIM_TASK_NAVIGATION) {  // navigation.hpp:55-75
        const double gm = y.navigation_goal_margin;
        const double xmin = -hw + gm, xmax = hw - gm, ymin = -hh + gm, ymax = hh - gm;
        for (int i = 0; i < N; ++i) {
            bool placed = false;
            for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
                const double gx = rng.uniform(xmin, xmax);
                const double gy = rng.uniform(ymin, ymax);
                bool ok = true;
                for (int q = 0; q < i; ++q)
                    if (hypot(gx - o.tf[2 * q], gy - o.tf[2 * q + 1]) < y.navigation_goal_separation) {
                        ok = false;
                        break;
                    }
                if (ok) {
                    o.tf[2 * i] = gx;
                    o.tf[2 * i + 1] = gy;
                    placed = true;
                }
            }
            if (!placed) { *bad = i; return kErrGoals; }
        }
    } else if (TASK == MRSIM_TASK_PREDATOR_PREY) {  // predator_prey.hpp:48-66
        const double xmin = -hw + sm, xmax = hw - sm, ymin = -hh + sm, ymax = hh - sm;
        bool placed = false;
        for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
            const double px = rng.uniform(xmin, xmax);
            const double py = rng.uniform(ymin, ymax);
            bool ok = true;
            for (int q = 0; q < N; ++q)
                if (hypot(px - o.x[q], py - o.y[q]) < y.pp_prey_spawn_clearance) { ok = false; break; }
            if (ok) {
                o.tf[0] = px;
                o.tf[1] = py;
                placed = true;
            }
        }
        if (!placed) { *bad = 0; return kErrPrey; }
        o.ti[0] = 0;  // flash_timer
    } else if (TASK == MRSIM_TASK_DISCOVERY) {  // discovery.hpp:27-38
        const double lm = y.discovery_landmark_margin;
        for (int k = 0; k < y.discovery_num_landmarks; ++k) {
            o.tf[2 * k] = rng.uniform(-hw + lm, hw - lm);
            o.tf[2 * k + 1] = rng.uniform(-hh + lm, hh - lm);
        }
        o.ti[0] = 0;
        o.ti[1] = 0;
    } else if (TASK == MRSIM_TASK_RWARE) {  // rware.hpp:25-44
        const int S = y.rware_num_slots, shelves = y.rware_num_shelves;
        for (int sl = 0; sl < S; ++sl) ti_set_byte(o.ti, sl, sl < shelves ? sl + 1 : 0);
        for (int i = 0; i < N; ++i) ti_set_byte(o.ti, S + i, 0);
        int pool[MRSIM_MAX_SLOTS];
        int np = 0;
        for (int i = 1; i <= shelves; ++i) pool[np++] = i;
        int nr = 0;
        for (int k = 0; k < y.rware_request_size && np > 0; ++k) {
            const int idx = static_cast<int>(rng.uniform_int(static_cast<uint64_t>(np)));
            ti_set_byte(o.ti, S + N + nr, pool[idx]);
            ++nr;
            for (int q = idx; q < np - 1; ++q) pool[q] = pool[q + 1];
            --np;
        }
    } else if (TASK == MRSIM_TASK_FORAGING) {  // foraging.hpp:27-49
        double l0 = -1e300, l1 = -1e300;  // two highest robot levels
        for (int i = 0; i < c.het_rows; ++i) {
            const double v = c.het[i][0];
            if (v > l0) { l1 = l0; l0 = v; }
            else if (v > l1) { l1 = v; }
        }
        const double top2 = l0 + (c.het_rows > 1 ? l1 : 0.0);
        int max_level = static_cast<int>(top2);
        if (max_level < 1) max_level = 1;
        const double rm = y.foraging_resource_margin;
        for (int r = 0; r < y.foraging_num_resources; ++r) {
            o.tf[2 * r] = rng.uniform(-hw + rm, hw - rm);
            o.tf[2 * r + 1] = rng.uniform(-hh + rm, hh - rm);
            o.ti[1 + r] = 1 + static_cast<int>(rng.uniform_int(static_cast<uint64_t>(max_level)));
        }
        o.ti[0] = 0;
    } else if (TASK == MRSIM_TASK_MATERIAL_TRANSPORT) {  // material_transport.hpp:28-40
        // normal(mean, sd) = mean + sd * normal() (rng.hpp:66)
        const double cn = __dadd_rn(y.mt_circle_mean, __dmul_rn(sqrt(y.mt_circle_variance), rng.normal()));
        const double circle = fmax(0.0, round(cn));
        const double rn = __dadd_rn(y.mt_rect_mean, __dmul_rn(sqrt(y.mt_rect_variance), rng.normal()));
        const double rect = fmax(0.0, round(rn));
        o.tf[0] = circle;
        o.tf[1] = rect;
        o.tf[2] = 0.0;            // delivered
        o.tf[3] = circle + rect;  // total_initial
        for (int i = 0; i < N; ++i) o.tf[4 + i] = 0.0;
    } else if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {  // arctic_transport.hpp:30-45
        const int cols = y.arctic_grid_cols, rows = y.arctic_grid_rows;
        for (int t = 0; t < cols * rows; ++t) ti_set_byte(o.ti, t, 0);
        for (int r = 0; r < rows; ++r)
            for (int cc = y.arctic_ground_cols_left; cc < cols - y.arctic_ground_cols_right; ++cc)
                ti_set_byte(o.ti, r * cols + cc, rng.uniform_int(2) == 0 ? 1 : 2);
    } else if (TASK == MRSIM_TASK_WAREHOUSE) {
        o.ti[0] = 0;
    } else if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {  // random_waypoints.hpp:29-37
        for (int i = 0; i < N; ++i) rwp_draw(c, rng, o.tf[2 * i], o.tf[2 * i + 1], o.tf[2 * N + i]);
    }
    return 0;
}


// ---------------------------------------------------------------------------
// One env's staged state during a step (shared memory of the group).
// ---------------------------------------------------------------------------
template <class Real>
struct EnvView {
    Real* xs;
    Real* ys;
    Real* ts;
    Real* tf;
    int* ti;
    int N;
    const int* drones;  // arctic: robot index of the k-th drone (robot-index order), else unused
    const double* prey_off;  // predator_prey: 8 candidate offsets (x, y), else unused
    const int* dcell = nullptr;  // arctic: (col, row) of the k-th drone, cached per env (or null)
    const double* het_flat = nullptr;  // full-team het_augment values in feature order (or null)
};

// arctic: the grid cell under a robot, with the observation's truncating casts
// (arctic_transport.hpp:108-112); used per drone for its 3x3 patch.
template <class Real>
__device__ __forceinline__ void arctic_cell(const mrsim_cfg& c, Real x, Real y, int& c0, int& r0) {
    const int cols = c.layout.arctic_grid_cols, rows = c.layout.arctic_grid_rows;
    const Real hw = Real(c.arena_half_width), hh = Real(c.arena_half_height);
    const Real cw = (hw - (-hw)) / Real(cols);
    const Real ch = (hh - (-hh)) / Real(rows);
    c0 = static_cast<int>(dclamp((x - (-hw)) / cw, Real(0), Real(cols - 1)));
    r0 = static_cast<int>(dclamp((y - (-hh)) / ch, Real(0), Real(rows - 1)));
}

// predator_prey: prey_step = agility * max step size (predator_prey.hpp:68-72) and the
// 8 compass offsets Vec2{cos(ang), sin(ang)} * prey_step, ang = (k-1) pi/4 (predator_prey.hpp:19-24)
inline void prey_offsets(const mrsim_cfg& c, double* out16) {
    double robot_step = 0.0;
    for (int i = 0; i < c.num_robots; ++i) robot_step = robot_step < c.step_sizes[i] ? c.step_sizes[i] : robot_step;
    const double prey_step = c.layout.pp_prey_agility * robot_step;
    for (int k = 1; k < 9; ++k) {
        const double ang = (k - 1) * (3.14159265358979323846 / 4.0);
        out16[2 * (k - 1)] = std::cos(ang) * prey_step;
        out16[2 * (k - 1) + 1] = std::sin(ang) * prey_step;
    }
}

// arctic drone list (het row [1,0,0]) in robot-index order; returns the count
__host__ __device__ inline int arctic_drones(const mrsim_cfg& c, int* out) {
    int nd = 0;
    for (int i = 0; i < c.num_robots; ++i)
        if (c.het[i][0] == 1.0) out[nd++] = i;
    return nd;
}

// ArcticTransportScenario::tile_at (arctic_transport.hpp:47-55): truncating
// casts, then clamp to the grid.
template <class Real>
__device__ __forceinline__ int arctic_tile_at(const mrsim_cfg& c, const int* ti, Real x, Real y) {
    const int cols = c.layout.arctic_grid_cols, rows = c.layout.arctic_grid_rows;
    const Real hw = Real(c.arena_half_width), hh = Real(c.arena_half_height);
    const Real cw = (hw - (-hw)) / Real(cols);
    const Real ch = (hh - (-hh)) / Real(rows);
    int cc = static_cast<int>((x - (-hw)) / cw);
    int rr = static_cast<int>((y - (-hh)) / ch);
    cc = cc < 0 ? 0 : (cc > cols - 1 ? cols - 1 : cc);
    rr = rr < 0 ? 0 : (rr > rows - 1 ? rows - 1 : rr);
    return ti_byte(ti, rr * cols + cc);
}

// Scenario::step_sizes (scenario.hpp:150-152; arctic override
// arctic_transport.hpp:58-73) for robot i at its current position.
template <int TASK, class Real>
__device__ __forceinline__ Real step_size_of(const mrsim_cfg& c, const int* ti, int i, Real x, Real y) {
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {
        const mrsim_layout& L = c.layout;
        if (c.het[i][0] == 1.0) return Real(L.arctic_normal_step);  // drones
        const int tile = arctic_tile_at<Real>(c, ti, x, y);
        if (tile == 0) return Real(L.arctic_normal_step);
        const bool matches = (c.het[i][1] == 1.0 && tile == 2) || (c.het[i][2] == 1.0 && tile == 1);
        return Real(matches ? L.arctic_fast_step : L.arctic_slow_step);
    }
    return Real(c.step_sizes[i]);
}

// prey_heuristic (predator_prey.hpp:15-34): of the prey's 9 candidate moves (stay, then E, NE,
// N, ... scaled by prey_step; offsets precomputed on the host with the reference's libm) inside
// the arena, the one farthest from the nearest robot; strict `>`, so the first index wins ties.
template <class Real>
__device__ __forceinline__ void prey_heuristic_dev(const mrsim_cfg& c, const double* prey_off, Real px, Real py,
                                                   const Real* xs, const Real* ys, int N, Real& bx, Real& by) {
    const Real hw = Real(c.arena_half_width), hh = Real(c.arena_half_height);
    bx = px;
    by = py;
    Real best = -Consts<Real>::inf;
    for (int k = 0; k < 9; ++k) {
        Real cx = px, cy = py;
        if (k > 0) {
            cx = px + Real(prey_off[2 * (k - 1)]);
            cy = py + Real(prey_off[2 * (k - 1) + 1]);
        }
        if (!(cx >= -hw && cx <= hw && cy >= -hh && cy <= hh)) continue;
        Real nearest = Consts<Real>::inf;
        for (int i = 0; i < N; ++i) nearest = dmin(nearest, dhypot(cx - xs[i], cy - ys[i]));
        if (nearest > best) {
            best = nearest;
            bx = cx;
            by = cy;
        }
    }
}

// Scenario::transition + Scenario::finalize, run by one lane on the staged
// state after the physics ticks. Returns the team reward (before the
// collision violation term, which the engine adds: batch.hpp:213-217).
template <int TASK, class Real>
__device__ Real transition_task(const mrsim_cfg& c, EnvView<Real>& v, Rng& rng, Real& metric) {
    const int N = v.N;
    const mrsim_layout& L = c.layout;
    if (TASK == MRSIM_TASK_NAVIGATION) {  // navigation.hpp:45-51
        Real total = 0;
        for (int i = 0; i < N; ++i) total += dhypot(v.xs[i] - v.tf[2 * i], v.ys[i] - v.tf[2 * i + 1]);
        return Real(c.coef[MRSIM_COEF_DIST]) * total;
    } else if (TASK == MRSIM_TASK_PREDATOR_PREY) {  // predator_prey.hpp:15-34, 74-91
        Real bx, by;
        prey_heuristic_dev<Real>(c, v.prey_off, v.tf[0], v.tf[1], v.xs, v.ys, N, bx, by);
        v.tf[0] = bx;
        v.tf[1] = by;
        bool tagged = false;
        for (int i = 0; i < N; ++i) tagged = tagged || dhypot(v.xs[i] - bx, v.ys[i] - by) <= Real(L.pp_tag_radius);
        if (tagged) {
            metric += Real(1);
            v.ti[0] = L.pp_flash_steps;
        } else if (v.ti[0] > 0) {
            v.ti[0] -= 1;
        }
        return tagged ? Real(c.coef[MRSIM_COEF_TAG]) : Real(0);
    } else if (TASK == MRSIM_TASK_DISCOVERY) {  // discovery.hpp:40-69
        const int K = L.discovery_num_landmarks;
        int sensed = v.ti[0], tagged = v.ti[1];
        int newly_sensed = 0, newly_tagged = 0;
        for (int k = 0; k < K; ++k) {
            if ((tagged >> k) & 1) continue;
            bool sense_hit = false, tag_hit = false;
            for (int i = 0; i < N; ++i) {
                const Real d = dhypot(v.xs[i] - v.tf[2 * k], v.ys[i] - v.tf[2 * k + 1]);
                const Real c0 = Real(c.het[i][0]), c1 = Real(c.het[i][1]);
                if (c0 > Real(0) && d <= c0) sense_hit = true;
                if (c1 > Real(0) && d <= c1) tag_hit = true;
            }
            if (sense_hit && !((sensed >> k) & 1)) {
                sensed |= 1 << k;
                ++newly_sensed;
            }
            if (tag_hit) {
                tagged |= 1 << k;
                ++newly_tagged;
            }
        }
        v.ti[0] = sensed;
        v.ti[1] = tagged;
        const bool all_tagged = tagged == ((K >= 32) ? -1 : ((1 << K) - 1));
        metric += Real(newly_tagged);
        return Real(c.coef[MRSIM_COEF_SENSE]) * Real(newly_sensed) + Real(c.coef[MRSIM_COEF_TAG]) * Real(newly_tagged) +
               Real(c.coef[MRSIM_COEF_STEP]) * (all_tagged ? Real(0) : Real(1));
    } else if (TASK == MRSIM_TASK_RWARE) {  // rware.hpp:70-107 (sequential over robots)
        const int S = L.rware_num_slots, R = rware_requests(L), shelves = L.rware_num_shelves;
        const Real half = Real(L.rware_slot_half);
        Real reward = 0;
        for (int i = 0; i < N; ++i) {
            const Real px = v.xs[i], py = v.ys[i];
            const int carried = ti_byte(v.ti, S + i);
            if (carried != 0 && rect_contains<Real>(L.rware_dropoff_zone, px, py)) {
                int it = -1;
                for (int q = 0; q < R; ++q)
                    if (ti_byte(v.ti, S + N + q) == carried) { it = q; break; }
                if (it >= 0) {
                    reward += Real(c.coef[MRSIM_COEF_DROPOFF]);
                    metric += Real(1);
                    int cand[MRSIM_MAX_SLOTS];
                    int nc = 0;
                    for (int id = 1; id <= shelves; ++id) {
                        bool req = false;
                        for (int q = 0; q < R; ++q) req = req || ti_byte(v.ti, S + N + q) == id;
                        if (!req) cand[nc++] = id;
                    }
                    if (nc > 0) ti_set_byte(v.ti, S + N + it, cand[rng.uniform_int(static_cast<uint64_t>(nc))]);
                }
                continue;
            }
            int slot = -1;  // slot_at (rware.hpp:46-52)
            for (int sl = 0; sl < S; ++sl) {
                if (dabs(px - Real(L.rware_slots[2 * sl])) <= half && dabs(py - Real(L.rware_slots[2 * sl + 1])) <= half) {
                    slot = sl;
                    break;
                }
            }
            if (slot < 0) continue;
            const int shelf = ti_byte(v.ti, slot);
            if (carried == 0 && shelf != 0) {
                ti_set_byte(v.ti, S + i, shelf);
                ti_set_byte(v.ti, slot, 0);
            } else if (carried != 0 && shelf == 0) {
                ti_set_byte(v.ti, slot, carried);
                ti_set_byte(v.ti, S + i, 0);
            }
        }
        return reward;
    } else if (TASK == MRSIM_TASK_FORAGING) {  // foraging.hpp:51-70
        const int M = L.foraging_num_resources;
        const Real radius = Real(L.foraging_radius);
        Real reward = 0;
        int foraged = v.ti[0];
        for (int r = 0; r < M; ++r) {
            if ((foraged >> r) & 1) continue;
            Real level_sum = 0;
            for (int i = 0; i < N; ++i)
                if (dhypot(v.xs[i] - v.tf[2 * r], v.ys[i] - v.tf[2 * r + 1]) <= radius) level_sum += Real(c.het[i][0]);
            const int level = v.ti[1 + r];
            if (level_sum >= Real(level)) {
                foraged |= 1 << r;
                reward += Real(c.coef[MRSIM_COEF_FORAGE]) * Real(level);
                metric += Real(1);
            }
        }
        v.ti[0] = foraged;
        return reward;
    } else if (TASK == MRSIM_TASK_MATERIAL_TRANSPORT) {  // material_transport.hpp:42-74 (sequential)
        Real circle = v.tf[0], rect = v.tf[1], delivered = v.tf[2];
        Real loaded = 0, dropped = 0;
        const Real ccx = Real(L.mt_circle_zone[0]), ccy = Real(L.mt_circle_zone[1]), cr = Real(L.mt_circle_zone[2]);
        for (int i = 0; i < N; ++i) {
            const Real px = v.xs[i], py = v.ys[i];
            const Real capacity = Real(c.het[i][1]);
            Real load = v.tf[4 + i];
            if (load > Real(0) && rect_contains<Real>(L.mt_dropoff_zone, px, py)) {
                dropped += load;
                delivered += load;
                load = 0;
            } else if (load == Real(0)) {
                if (dhypot(ccx - px, ccy - py) <= cr && circle > Real(0)) {
                    const Real take = dmin(capacity, circle);
                    circle -= take;
                    load = take;
                    loaded += take;
                } else if (rect_contains<Real>(L.mt_rect_zone, px, py) && rect > Real(0)) {
                    const Real take = dmin(capacity, rect);
                    rect -= take;
                    load = take;
                    loaded += take;
                }
            }
            v.tf[4 + i] = load;
        }
        v.tf[0] = circle;
        v.tf[1] = rect;
        v.tf[2] = delivered;
        metric = circle + rect;
        const bool zones_empty = circle == Real(0) && rect == Real(0);
        return Real(c.coef[MRSIM_COEF_LOAD]) * loaded + Real(c.coef[MRSIM_COEF_DROPOFF]) * dropped +
               Real(c.coef[MRSIM_COEF_STEP]) * (zones_empty ? Real(0) : Real(1));
    } else if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {  // arctic_transport.hpp:75-86
        const double* gz = L.arctic_goal_zone;
        Real summed = 0;
        bool all_in = true;
        for (int i = 0; i < N; ++i) {
            if (c.het[i][0] == 1.0) continue;
            const Real px = v.xs[i], py = v.ys[i];
            const Real dx = dmax(dmax(Real(gz[0]) - px, Real(0)), px - Real(gz[1]));
            const Real dy = dmax(dmax(Real(gz[2]) - py, Real(0)), py - Real(gz[3]));
            summed += dhypot(dx, dy);
            all_in = all_in && rect_contains<Real>(gz, px, py);
        }
        return Real(c.coef[MRSIM_COEF_DIST]) * summed + Real(c.coef[MRSIM_COEF_STEP]) * (all_in ? Real(0) : Real(1));
    } else if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {  // random_waypoints.hpp:52-66 (sequential over robots)
        const Real tol = Real(L.rwp_arrival_tolerance);
        for (int i = 0; i < N; ++i) {
            Real cx = v.xs[i], cy = v.ys[i];
            if (c.controller == MRSIM_CONTROLLER_UNICYCLE_POSITION) {  // projected_point (controllers.hpp:34-36)
                Real sn, cs;
                dsincos(v.ts[i], &sn, &cs);
                cx = v.xs[i] + cs * Real(c.projection_distance);
                cy = v.ys[i] + sn * Real(c.projection_distance);
            }
            if (dhypot(cx - v.tf[2 * i], cy - v.tf[2 * i + 1]) <= tol) {
                double tx, ty, th;
                rwp_draw(c, rng, tx, ty, th);
                v.tf[2 * i] = Real(tx);
                v.tf[2 * i + 1] = Real(ty);
                v.tf[2 * N + i] = Real(th);
            }
        }
        return Real(0);
    } else {  // warehouse.hpp:36-54
        Real reward = 0;
        int loaded = v.ti[0];
        for (int i = 0; i < N; ++i) {
            const Real px = v.xs[i], py = v.ys[i];
            const bool green = c.het[i][0] == 1.0;
            const double* pickup = green ? L.warehouse_green_right : L.warehouse_red_right;
            const double* deliver = green ? L.warehouse_green_left : L.warehouse_red_left;
            const bool is_loaded = (loaded >> i) & 1;
            if (!is_loaded && rect_contains<Real>(pickup, px, py)) {
                loaded |= 1 << i;
                reward += Real(c.coef[MRSIM_COEF_LOAD]);
            } else if (is_loaded && rect_contains<Real>(deliver, px, py)) {
                loaded &= ~(1 << i);
                reward += Real(c.coef[MRSIM_COEF_DELIVERY]);
                metric += Real(1);
            }
        }
        v.ti[0] = loaded;
        return reward;
    }
}

// Scenario::finalize (navigation.hpp:53-61, arctic_transport.hpp:88-97).
template <int TASK, class Real>
__device__ void finalize_task(const mrsim_cfg& c, const EnvView<Real>& v, Real& metric, int& success) {
    if (TASK == MRSIM_TASK_NAVIGATION) {
        bool all_on = true;
        for (int i = 0; i < v.N; ++i)
            all_on = all_on && dhypot(v.xs[i] - v.tf[2 * i], v.ys[i] - v.tf[2 * i + 1]) <= Real(c.layout.navigation_on_goal_radius);
        success = all_on ? 1 : 0;
        metric = all_on ? Real(1) : Real(0);
    } else if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {
        bool all_in = true;
        for (int i = 0; i < v.N; ++i) {
            if (c.het[i][0] == 1.0) continue;
            all_in = all_in && rect_contains<Real>(c.layout.arctic_goal_zone, v.xs[i], v.ys[i]);
        }
        success = all_in ? 1 : 0;
        metric = all_in ? Real(1) : Real(0);
    }
}

// Observation dimension before/after het_augment.
__host__ __device__ inline int base_obs_dim(const mrsim_cfg& c) {
    const int N = c.num_robots;
    const mrsim_layout& L = c.layout;
    const int base = 3 + 2 * (N - 1);
    switch (c.task) {
        case MRSIM_TASK_NAVIGATION: return 5;
        case MRSIM_TASK_PREDATOR_PREY: return base + 2;
        case MRSIM_TASK_DISCOVERY: return base + 2 * L.discovery_num_landmarks;
        case MRSIM_TASK_RWARE: return base + 3 * L.rware_num_slots + rware_requests(L) + 1;
        case MRSIM_TASK_FORAGING: return base + 3 * L.foraging_num_resources;
        case MRSIM_TASK_MATERIAL_TRANSPORT: return base + 3;
        case MRSIM_TASK_ARCTIC_TRANSPORT: {
            int drones = 0;
            for (int i = 0; i < N; ++i) drones += (c.het[i][0] == 1.0) ? 1 : 0;
            return base + 1 + 9 * drones;
        }
        case MRSIM_TASK_WAREHOUSE: return base + 1;
        case MRSIM_TASK_RANDOM_WAYPOINTS: return 5;
        default: return 0;
    }
}
__host__ __device__ inline int obs_dim_of(const mrsim_cfg& c) {
    int d = base_obs_dim(c);
    if (c.het_obs_mode == MRSIM_HET_OBS_OWN) d += c.het_cols;
    else if (c.het_obs_mode == MRSIM_HET_OBS_FULL_TEAM) d += c.het_rows * c.het_cols;
    return d;
}

// Feature q of robot r's observation, in the state's precision (stores
// round it to fp32; the on-device policy consumes it unrounded): Scenario::observe + base_observation
// (scenario.hpp:200-210) + het_augment (framework.hpp:61-76).
template <int TASK, class Real>
__device__ Real obs_feature(const mrsim_cfg& c, const EnvView<Real>& v, int r, int q, int bdim) {
    const int N = v.N;
    const mrsim_layout& L = c.layout;
    if (q >= bdim) {  // het_augment
        const int k = q - bdim;
        if (c.het_obs_mode == MRSIM_HET_OBS_OWN) return Real(c.het[r][k]);
        if (v.het_flat) return Real(v.het_flat[k]);
        return Real(c.het[k / c.het_cols][k % c.het_cols]);
    }
    if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {  // random_waypoints.hpp:70-76: own pose + target
        switch (q) {
            case 0: return Real(v.xs[r]);
            case 1: return Real(v.ys[r]);
            case 2: return Real(v.ts[r]);
            case 3: return Real(v.tf[2 * r]);
            default: return Real(v.tf[2 * r + 1]);
        }
    }
    if (TASK == MRSIM_TASK_NAVIGATION) {  // navigation.hpp:64-70
        switch (q) {
            case 0: return Real(v.xs[r]);
            case 1: return Real(v.ys[r]);
            case 2: return Real(v.ts[r]);
            case 3: return Real(v.tf[2 * r] - v.xs[r]);
            default: return Real(v.tf[2 * r + 1] - v.ys[r]);
        }
    }
    const int base = 3 + 2 * (N - 1);
    if (q < base) {
        if (q == 0) return Real(v.xs[r]);
        if (q == 1) return Real(v.ys[r]);
        if (q == 2) return Real(v.ts[r]);
        const int k = (q - 3) >> 1;
        const int j = k < r ? k : k + 1;
        return Real(((q - 3) & 1) ? v.ys[j] : v.xs[j]);
    }
    const int f = q - base;
    if (TASK == MRSIM_TASK_PREDATOR_PREY) return Real(v.tf[f]);
    if (TASK == MRSIM_TASK_DISCOVERY) {  // discovery.hpp:71-82
        const int k = f >> 1;
        const bool visible = ((v.ti[0] >> k) & 1) && !((v.ti[1] >> k) & 1);
        return Real(visible ? double(v.tf[f]) : L.discovery_sentinel[f & 1]);
    }
    if (TASK == MRSIM_TASK_RWARE) {  // rware.hpp:111-124
        const int S = L.rware_num_slots;
        if (f < 3 * S) {
            const int sl = f / 3, comp = f % 3;
            if (comp < 2) return Real(L.rware_slots[2 * sl + comp]);
            return Real(ti_byte(v.ti, sl));
        }
        const int g2 = f - 3 * S;
        if (g2 < rware_requests(L)) return Real(ti_byte(v.ti, S + N + g2));
        return Real(ti_byte(v.ti, S + r));
    }
    if (TASK == MRSIM_TASK_FORAGING) {  // foraging.hpp:72-84
        const int rr = f / 3, comp = f % 3;
        const bool live = !((v.ti[0] >> rr) & 1);
        if (comp < 2) return Real(live ? double(v.tf[2 * rr + comp]) : L.discovery_sentinel[comp]);
        return live ? Real(v.ti[1 + rr]) : Real(0);
    }
    if (TASK == MRSIM_TASK_MATERIAL_TRANSPORT) {  // material_transport.hpp:77-85
        if (f == 0) return Real(v.tf[4 + r]);
        return Real(v.tf[f - 1]);  // 1 -> circle (tf[0]), 2 -> rect (tf[1])
    }
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {  // arctic_transport.hpp:102-123
        if (f == 0) return Real(arctic_tile_at<Real>(c, v.ti, v.xs[r], v.ys[r]));
        const int g2 = f - 1;
        const int which = g2 / 9, cell = g2 % 9;
        const int cols = L.arctic_grid_cols, rows = L.arctic_grid_rows;
        int c0, r0;
        if (v.dcell) {
            c0 = v.dcell[2 * which];
            r0 = v.dcell[2 * which + 1];
        } else {
            const int d = v.drones[which];  // which-th drone in robot-index order
            arctic_cell<Real>(c, v.xs[d], v.ys[d], c0, r0);
        }
        const int rr = r0 + cell / 3 - 1, cc = c0 + cell % 3 - 1;
        const bool in = rr >= 0 && rr < rows && cc >= 0 && cc < cols;
        return in ? Real(ti_byte(v.ti, rr * cols + cc)) : Real(0);
    }
    // warehouse.hpp:57-63
    return ((v.ti[0] >> r) & 1) ? Real(1) : Real(0);
}

}  // namespace mrsim_dev
