// scripted.cuh — the reference's scripted policies on the device (SURVEY.md
// 8(f) row 4): PolicyKind::ScriptedGoal (grid BFS planner toward the task's
// scripted goal, policy.hpp:242-360 + Scenario::scripted_goal) and
// PolicyKind::PreyChaser (policy.hpp:362-416), producing the step's actions.
//
// One warp per environment, robots in turn. The planner's occupancy grid
// (0.05 m cells over the arena) is a bitset built with one ballot per 32
// cells; the BFS from the goal is level-synchronous (each level marks the
// free, unvisited cells with a neighbour in the frontier bitset), which yields
// exactly the reference's queue-BFS distances (shortest 8-connected path
// lengths, whatever the queue order); the subgoal walk
// and the action scoring then run on one lane in the reference's order.
// Geometry uses explicitly rounded multiply/add where the reference's
// expression would otherwise be contracted into an FMA; hypot comes from the
// device libm (<= 1 ulp from glibc), so a blocked-cell or score decision can
// flip only at a near-tie.
#pragma once

#include <cstddef>

#include "policy.cuh"

namespace mrsim_dev {

constexpr int kGridMaxCells = 4096;  // 0.05 m cells: up to a 3.2 x 3.2 m arena
constexpr int kGridWords = kGridMaxCells / 32;

struct ScriptedSmem {
    double xs[MRSIM_MAX_ROBOTS], ys[MRSIM_MAX_ROBOTS], ts[MRSIM_MAX_ROBOTS], tf[kTfMax];
    int ti[kTiMax];
    int drones[MRSIM_MAX_ROBOTS];
    unsigned blocked[kGridWords], frontier[kGridWords], visited[kGridWords], next[kGridWords];
    unsigned colE[kGridWords], colW[kGridWords];  // cells that have an east / west neighbour column
    unsigned short dist[kGridMaxCells];  // BFS level + 1 (0 = unreached); last: see scripted_smem_stride
};

// Per-warp shared-memory footprint for an arena of `cells` planner cells: `dist` (the last member)
// is cut to the grid's whole 32-cell words, so a 3.2 x 2 m arena (2,560 cells) takes 9.2 KB instead
// of 12.2 KB per warp and six 4-warp blocks fit an SM (registers allow six; the full struct, four).
__host__ __device__ constexpr int scripted_smem_stride(int cells) {
    return (static_cast<int>(offsetof(ScriptedSmem, dist)) + ((cells + 31) / 32) * 32 * 2 + 15) / 16 * 16;
}

struct Vec2d {
    double x, y;
};

__device__ __forceinline__ double dist2d(double ax, double ay, double bx, double by) { return hypot(ax - bx, ay - by); }

// Scenario::scripted_goal of every task (scenarios/*.hpp), for robot r.
template <int TASK>
__device__ Vec2d scripted_goal_dev(const mrsim_cfg& c, const ScriptedSmem& s, int r) {
    const mrsim_layout& y = c.layout;
    const int N = c.num_robots;
    const double sx = s.xs[r], sy = s.ys[r];
    auto rect_center = [](const double* q) { return Vec2d{0.5 * (q[0] + q[1]), 0.5 * (q[2] + q[3])}; };
    if (TASK == MRSIM_TASK_NAVIGATION) return Vec2d{s.tf[2 * r], s.tf[2 * r + 1]};  // navigation.hpp:72-74
    if (TASK == MRSIM_TASK_PREDATOR_PREY) return Vec2d{s.tf[0], s.tf[1]};           // predator_prey.hpp:102-104
    if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) return Vec2d{s.tf[2 * r], s.tf[2 * r + 1]};
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) return rect_center(y.arctic_goal_zone);  // arctic_transport.hpp:125-127
    if (TASK == MRSIM_TASK_WAREHOUSE) {  // warehouse.hpp:65-72
        const bool green = c.het[r][0] == 1.0;
        const bool loaded = (s.ti[0] >> r) & 1;
        if (loaded) return rect_center(green ? y.warehouse_green_left : y.warehouse_red_left);
        return rect_center(green ? y.warehouse_green_right : y.warehouse_red_right);
    }
    if (TASK == MRSIM_TASK_MATERIAL_TRANSPORT) {  // material_transport.hpp:87-94
        if (s.tf[4 + r] > 0.0) return rect_center(y.mt_dropoff_zone);
        if (s.tf[0] > 0.0) return Vec2d{y.mt_circle_zone[0], y.mt_circle_zone[1]};
        if (s.tf[1] > 0.0) return rect_center(y.mt_rect_zone);
        return Vec2d{sx, sy};
    }
    Vec2d best{sx, sy};
    double best_d = Consts<double>::inf;
    if (TASK == MRSIM_TASK_DISCOVERY) {  // discovery.hpp:84-98: nearest untagged landmark
        for (int k = 0; k < y.discovery_num_landmarks; ++k) {
            if ((s.ti[1] >> k) & 1) continue;
            const double d = dist2d(sx, sy, s.tf[2 * k], s.tf[2 * k + 1]);
            if (d < best_d) {
                best_d = d;
                best = Vec2d{s.tf[2 * k], s.tf[2 * k + 1]};
            }
        }
        return best;
    }
    if (TASK == MRSIM_TASK_FORAGING) {  // foraging.hpp:86-100: nearest unforaged resource
        for (int k = 0; k < y.foraging_num_resources; ++k) {
            if ((s.ti[0] >> k) & 1) continue;
            const double d = dist2d(sx, sy, s.tf[2 * k], s.tf[2 * k + 1]);
            if (d < best_d) {
                best_d = d;
                best = Vec2d{s.tf[2 * k], s.tf[2 * k + 1]};
            }
        }
        return best;
    }
    if (TASK == MRSIM_TASK_RWARE) {  // rware.hpp:126-158
        const int S = y.rware_num_slots, R = rware_requests(y);
        auto requested = [&](int shelf) {
            for (int q = 0; q < R; ++q)
                if (ti_byte(s.ti, S + N + q) == shelf) return true;
            return false;
        };
        const int carried = ti_byte(s.ti, S + r);
        if (carried != 0) {
            if (requested(carried)) return rect_center(y.rware_dropoff_zone);
            for (int i = 0; i < S; ++i) {  // nearest empty slot
                if (ti_byte(s.ti, i) != 0) continue;
                const double d = dist2d(sx, sy, y.rware_slots[2 * i], y.rware_slots[2 * i + 1]);
                if (d < best_d) {
                    best_d = d;
                    best = Vec2d{y.rware_slots[2 * i], y.rware_slots[2 * i + 1]};
                }
            }
            return best;
        }
        for (int i = 0; i < S; ++i) {  // nearest staged, requested shelf
            const int shelf = ti_byte(s.ti, i);
            if (shelf == 0 || !requested(shelf)) continue;
            const double d = dist2d(sx, sy, y.rware_slots[2 * i], y.rware_slots[2 * i + 1]);
            if (d < best_d) {
                best_d = d;
                best = Vec2d{y.rware_slots[2 * i], y.rware_slots[2 * i + 1]};
            }
        }
        return best;
    }
    return best;
}

// action_direction (framework.hpp:80-94): stay, +y, -y, -x, +x
__device__ __forceinline__ void action_dir(int a, double& dx, double& dy) {
    dx = (a == 3) ? -1.0 : ((a == 4) ? 1.0 : 0.0);
    dy = (a == 1) ? 1.0 : ((a == 2) ? -1.0 : 0.0);
}

// Where the robot can be at the end of this step toward action a's waypoint
// (policy.hpp:203-235, 350-356): min(travel, |wp - self|) along the waypoint direction.
__device__ __forceinline__ Vec2d reached_point(const mrsim_cfg& c, double sx, double sy, int a, double step,
                                              double travel) {
    double dx, dy;
    action_dir(a, dx, dy);
    double wx = __dadd_rn(sx, __dmul_rn(dx, step)), wy = __dadd_rn(sy, __dmul_rn(dy, step));
    wx = dclamp(wx, -c.arena_half_width, c.arena_half_width);
    wy = dclamp(wy, -c.arena_half_height, c.arena_half_height);
    const double tx = wx - sx, ty = wy - sy;
    const double len = hypot(tx, ty);
    Vec2d rp{sx, sy};
    if (len > 1e-12) {
        const double f = dmin(travel, len) / len;
        rp = Vec2d{__dadd_rn(sx, __dmul_rn(tx, f)), __dadd_rn(sy, __dmul_rn(ty, f))};
    }
    return rp;
}

// argmin_action_toward (policy.hpp:203-235): the first action whose reached point is nearest.
__device__ __forceinline__ int argmin_action_toward(const mrsim_cfg& c, double sx, double sy, Vec2d target,
                                                    double step, double travel) {
    int best = 0;
    double best_d = Consts<double>::inf;
    for (int a = 0; a < 5; ++a) {
        const Vec2d rp = reached_point(c, sx, sy, a, step, travel);
        const double d = dist2d(rp.x, rp.y, target.x, target.y);
        if (d < best_d) {
            best_d = d;
            best = a;
        }
    }
    return best;
}

// prey_chaser_action (policy.hpp:370-416)
__device__ inline int prey_chaser_dev(const mrsim_cfg& c, const ScriptedSmem& s, const double* prey_off, int robot,
                               double travel) {
    const int N = c.num_robots;
    const double hw = c.arena_half_width, hh = c.arena_half_height;
    const double px = s.tf[0], py = s.tf[1];
    const double sx = px >= 0 ? 1.0 : -1.0, sy = py >= 0 ? 1.0 : -1.0;
    const Vec2d corner{sx * hw, sy * hh};
    int driver = 0;
    double best_d = Consts<double>::inf;
    for (int j = 0; j < N; ++j) {
        const double d = dist2d(s.xs[j], s.ys[j], px, py);
        if (d < best_d) {
            best_d = d;
            driver = j;
        }
    }
    Vec2d target;
    const double corner_dist = dist2d(px, py, corner.x, corner.y);
    if (corner_dist < 0.7) {  // squeeze: the prey's next position
        double bx, by;
        prey_heuristic_dev<double>(c, prey_off, px, py, s.xs, s.ys, N, bx, by);
        target = Vec2d{bx, by};
    } else if (robot == driver) {  // pressure from the side opposite the corner
        const double inv = 1.0 / corner_dist;
        const double ddx = __dmul_rn(corner.x - px, inv), ddy = __dmul_rn(corner.y - py, inv);
        target = Vec2d{px - __dmul_rn(ddx, 0.15), py - __dmul_rn(ddy, 0.15)};
    } else {  // stations on the two escape routes
        int slot = 0;
        for (int j = 0; j < N; ++j) {
            if (j == driver) continue;
            if (j == robot) break;
            ++slot;
        }
        const double reach = __dadd_rn(0.55, __dmul_rn(0.35, static_cast<double>(slot / 2)));
        // along_x = (-sx, 0), along_y = (0, -sy)
        if (slot % 2 == 0)
            target = Vec2d{__dadd_rn(__dadd_rn(corner.x, __dmul_rn(-sx, reach)), 0.0 * 0.14),
                           __dadd_rn(__dadd_rn(corner.y, 0.0 * reach), __dmul_rn(-sy, 0.14))};
        else
            target = Vec2d{__dadd_rn(__dadd_rn(corner.x, 0.0 * reach), __dmul_rn(-sx, 0.14)),
                           __dadd_rn(__dadd_rn(corner.y, __dmul_rn(-sy, reach)), 0.0 * 0.14)};
    }
    target.x = dclamp(target.x, -hw, hw);
    target.y = dclamp(target.y, -hh, hh);
    return argmin_action_toward(c, s.xs[robot], s.ys[robot], target, c.step_sizes[robot], travel);
}

// scripted_goal_action (policy.hpp:242-360) for `robot`, run by the whole warp.
template <int TASK>
__device__ int scripted_goal_action_dev(const mrsim_cfg& c, ScriptedSmem& s, int robot, double step_size,
                                        double travel) {
    const int lane = threadIdx.x & 31;
    const int N = c.num_robots;
    const double xmin = -c.arena_half_width, xmax = c.arena_half_width;
    const double ymin = -c.arena_half_height, ymax = c.arena_half_height;
    const double robot_clear = c.safety_radius + 2.0 * c.projection_distance + 0.03;
    const double wall_clear = c.boundary_margin + c.projection_distance + 0.03;
    const double cell = 0.05;
    const int cols = static_cast<int>((xmax - xmin) / cell);
    const int rows = static_cast<int>((ymax - ymin) / cell);
    const int ncell = cols * rows, nw = (ncell + 31) / 32;
    const double sx = s.xs[robot], sy = s.ys[robot];
    const Vec2d goal = scripted_goal_dev<TASK>(c, s, robot);
    auto center = [&](int cc, int rr) {
        return Vec2d{__dadd_rn(xmin, __dmul_rn(cc + 0.5, cell)), __dadd_rn(ymin, __dmul_rn(rr + 0.5, cell))};
    };
    auto cell_of = [&](double x, double y, int& cc, int& rr) {
        cc = static_cast<int>(dclamp((x - xmin) / cell, 0.0, cols - 1.0));
        rr = static_cast<int>(dclamp((y - ymin) / cell, 0.0, rows - 1.0));
    };
    // occupancy (policy.hpp:263-274): one ballot per 32 cells
    for (int w = 0; w < nw; ++w) {
        const int idx = w * 32 + lane;
        bool b = false;
        if (idx < ncell) {
            const Vec2d p = center(idx % cols, idx / cols);
            b = p.x < xmin + wall_clear || p.x > xmax - wall_clear || p.y < ymin + wall_clear ||
                p.y > ymax - wall_clear;
            for (int j = 0; j < N && !b; ++j) {
                if (j == robot) continue;
                b = dist2d(p.x, p.y, s.xs[j], s.ys[j]) < robot_clear;
            }
        }
        const unsigned word = __ballot_sync(0xffffffffu, b || idx >= ncell);  // bits past the grid: never free
        const unsigned east = __ballot_sync(0xffffffffu, idx < ncell && idx % cols != cols - 1);
        const unsigned west = __ballot_sync(0xffffffffu, idx < ncell && idx % cols != 0);
        if (lane == 0) {
            s.blocked[w] = word;
            s.colE[w] = east;
            s.colW[w] = west;
        }
    }
    __syncwarp();
    int sc, sr, gc, gr;
    cell_of(sx, sy, sc, sr);
    cell_of(goal.x, goal.y, gc, gr);
    if (lane == 0) s.blocked[(sr * cols + sc) >> 5] &= ~(1u << ((sr * cols + sc) & 31));  // start free by fiat
    __syncwarp();
    if ((s.blocked[(gr * cols + gc) >> 5] >> ((gr * cols + gc) & 31)) & 1u) {
        // blocked goal: the nearest free cell, first in row-major order on ties (policy.hpp:283-297)
        double bd = Consts<double>::inf;
        int bi = gr * cols + gc;
        for (int idx = lane; idx < ncell; idx += 32) {
            if ((s.blocked[idx >> 5] >> (idx & 31)) & 1u) continue;
            const Vec2d p = center(idx % cols, idx / cols);
            const double d = dist2d(p.x, p.y, goal.x, goal.y);
            if (d < bd) {
                bd = d;
                bi = idx;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double od = __shfl_xor_sync(0xffffffffu, bd, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (od < bd || (od == bd && oi < bi)) {
                bd = od;
                bi = oi;
            }
        }
        gc = bi % cols;
        gr = bi / cols;
    }
    // BFS from the goal (policy.hpp:299-318) as level-synchronous bitset expansion
    const int g0 = gr * cols + gc;
    for (int w = lane; w < nw; w += 32) {
        const unsigned gbit = (w == (g0 >> 5)) ? (1u << (g0 & 31)) : 0u;
        s.frontier[w] = gbit;
        s.visited[w] = gbit;
    }
    for (int idx = lane; idx < ncell; idx += 32) s.dist[idx] = (idx == g0) ? 1 : 0;
    __syncwarp();
    // 32 bits of a bitset starting at bit `start` (may lie outside the grid: those bits read as 0)
    auto window = [&](const unsigned* bs, int start) -> unsigned {
        const int wq = start >= 0 ? (start >> 5) : -((31 - start) >> 5);
        const int sh = start - wq * 32;
        const unsigned lo = (wq >= 0 && wq < nw) ? bs[wq] : 0u;
        const unsigned hi = (wq + 1 >= 0 && wq + 1 < nw) ? bs[wq + 1] : 0u;
        return sh ? ((lo >> sh) | (hi << (32 - sh))) : lo;
    };
    for (int level = 1; level < ncell; ++level) {
        // a free, unvisited cell joins this level if any of its 8 neighbours is in the frontier
        bool any = false;
        for (int w = lane; w < nw; w += 32) {
            const int base = w * 32;
            unsigned hit = 0u;
            hit |= window(s.frontier, base + 1) & s.colE[w];             // (+1, 0)
            hit |= window(s.frontier, base - 1) & s.colW[w];             // (-1, 0)
            hit |= window(s.frontier, base + cols);                      // (0, +1)
            hit |= window(s.frontier, base - cols);                      // (0, -1)
            hit |= window(s.frontier, base + cols + 1) & s.colE[w];      // (+1, +1)
            hit |= window(s.frontier, base - cols + 1) & s.colE[w];      // (+1, -1)
            hit |= window(s.frontier, base + cols - 1) & s.colW[w];      // (-1, +1)
            hit |= window(s.frontier, base - cols - 1) & s.colW[w];      // (-1, -1)
            const unsigned word = hit & ~s.visited[w] & ~s.blocked[w];
            s.next[w] = word;
            any = any || word != 0u;
        }
        __syncwarp();
        if (!__any_sync(0xffffffffu, any)) break;
        for (int w = lane; w < nw; w += 32) {
            const unsigned word = s.next[w];
            s.frontier[w] = word;
            s.visited[w] |= word;
            for (unsigned m = word; m; m &= m - 1) s.dist[w * 32 + __ffs(m) - 1] = static_cast<unsigned short>(level + 1);
        }
        __syncwarp();
    }
    int action = 0;
    if (lane == 0) {
        auto dist_at = [&](int cc, int rr) { return static_cast<int>(s.dist[rr * cols + cc]) - 1; };  // -1 unreached
        Vec2d subgoal = goal;
        const int d0 = dist_at(sc, sr);
        if (d0 > 0) {  // policy.hpp:320-340
            int cc = sc, rr = sr;
            for (int hop = 0; hop < 5; ++hop) {
                const int cur = dist_at(cc, rr);
                if (cur <= 0) break;
                for (int k = 0; k < 8; ++k) {
                    const int dc = (k == 0 || k == 4 || k == 5) ? 1 : ((k == 1 || k == 6 || k == 7) ? -1 : 0);
                    const int dr = (k == 2 || k == 4 || k == 6) ? 1 : ((k == 3 || k == 5 || k == 7) ? -1 : 0);
                    const int nc = cc + dc, nr = rr + dr;
                    if (nc < 0 || nr < 0 || nc >= cols || nr >= rows) continue;
                    const int nd = dist_at(nc, nr);
                    if (nd >= 0 && nd < cur) {
                        cc = nc;
                        rr = nr;
                        break;
                    }
                }
            }
            subgoal = center(cc, rr);
            if (d0 <= 5) subgoal = goal;
        }
        // score the actions (policy.hpp:342-359)
        double best_score = Consts<double>::inf;
        for (int a = 0; a < 5; ++a) {
            const Vec2d rp = reached_point(c, sx, sy, a, step_size, travel);
            double score = dist2d(rp.x, rp.y, subgoal.x, subgoal.y);
            for (int j = 0; j < N; ++j) {
                if (j == robot) continue;
                const double d_new = dist2d(rp.x, rp.y, s.xs[j], s.ys[j]);
                if (d_new < dist2d(sx, sy, s.xs[j], s.ys[j]) && d_new < robot_clear) score += robot_clear - d_new;
            }
            if (score < best_score) {
                best_score = score;
                action = a;
            }
        }
    }
    return __shfl_sync(0xffffffffu, action, 0);
}

template <class Real>
struct ScriptedParams {
    mrsim_cfg c;
    DevState<Real> s;
    long long B;
    int N, nf, ni;
    int kind;  // MRSIM_POLICY_SCRIPTED_GOAL / MRSIM_POLICY_PREY_CHASER
    double prey_off[16];
    int8_t* actions;
    unsigned* ticket;  // [2] env counters, used by alternate launches (serial & 1)
    long long serial;  // launch count of this context's scripted kernel
    int smem_stride;   // bytes of shared memory per warp (scripted_smem_stride)
    int num_sms;       // of the context's device (grid sizing)
};

template <class Real, int TASK>
__global__ void __launch_bounds__(32 * kPolicyWarps) scripted_kernel(const __grid_constant__ ScriptedParams<Real> p) {
    extern __shared__ __align__(16) unsigned char scr_smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    ScriptedSmem& sm = *reinterpret_cast<ScriptedSmem*>(scr_smem + wib * p.smem_stride);
    const mrsim_cfg& c = p.c;
    const int N = p.N;
    const double travel = c.si_max_speed * c.dt * c.sub_steps;  // policy.hpp:246
    // Dynamic env tasks (planner cost varies widely per env): a warp takes the next env from
    // counter serial & 1; this launch clears the other one for the next launch (stream order).
    if (MRSIM_DYN_SCHED && blockIdx.x == 0 && threadIdx.x == 0) p.ticket[(p.serial + 1) & 1] = 0u;
    auto next_env = [&](long long e_static) -> long long {
        if (!MRSIM_DYN_SCHED) return e_static;
        unsigned t = 0;
        if (lane == 0) t = atomicAdd(p.ticket + (p.serial & 1), 1u);
        return static_cast<long long>(__shfl_sync(0xffffffffu, t, 0));
    };
    const long long stride = static_cast<long long>(gridDim.x) * kPolicyWarps;
    for (long long e = next_env(static_cast<long long>(blockIdx.x) * kPolicyWarps + wib); e < p.B;
         e = next_env(e + stride)) {
        __syncwarp();
        if (lane < N) {
            sm.xs[lane] = double(p.s.px[e * N + lane]);
            sm.ys[lane] = double(p.s.py[e * N + lane]);
            sm.ts[lane] = double(p.s.pt[e * N + lane]);
        }
        for (int f = lane; f < p.nf; f += 32) sm.tf[f] = double(p.s.tf[static_cast<long long>(f) * p.B + e]);
        for (int w = lane; w < p.ni; w += 32) sm.ti[w] = p.s.ti[static_cast<long long>(w) * p.B + e];
        __syncwarp();
        if (TASK == MRSIM_TASK_PREDATOR_PREY && p.kind == MRSIM_POLICY_PREY_CHASER) {
            if (lane < N) p.actions[e * N + lane] = static_cast<int8_t>(prey_chaser_dev(c, sm, p.prey_off, lane, travel));
            continue;  // (the loop head syncs the warp before the next env is staged)
        }
        for (int r = 0; r < N; ++r) {
            int a;
            {
                const double step = double(step_size_of<TASK, double>(c, sm.ti, r, sm.xs[r], sm.ys[r]));
                a = scripted_goal_action_dev<TASK>(c, sm, r, step, travel);
            }
            if (lane == 0) p.actions[e * N + r] = static_cast<int8_t>(a);
            __syncwarp();
        }
    }
}

}  // namespace mrsim_dev
