/*
 * mrsim_oracle.c — TEST INFRASTRUCTURE: plain-C fp64 restatement of the
 * reference hot path. See mrsim_oracle.h. Paths in citations are relative
 * to /root/reference/proj/include/mrsim. Operation order follows the
 * reference expression by expression so that, compiled with the same flags
 * (no FMA contraction), results are bit-identical to the reference.
 */
#include "mrsim_oracle.h"

#include <math.h>
#include <stdio.h>
#include <string.h>

#define PI 3.14159265358979323846 /* core.hpp:16 */
#define MAXN MRSIM_MAX_ROBOTS
#define MAXV (2 * MAXN)
#define MAXROWS (MAXN * (MAXN - 1) / 2 + 4 * MAXN + MAXN * MRSIM_MAX_SLOTS + 2 * MAXV)

static int fail(char* err, int len, int code, const char* msg) {
    if (err && len > 0) {
        strncpy(err, msg, (size_t)len - 1);
        err[len - 1] = 0;
    }
    return code;
}

/* ---------------- RNG (rng.hpp:15-67, harness.hpp:25-34) ---------------- */

uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static const uint64_t GAMMA = 0x9E3779B97F4A7C15ULL;
uint64_t orc_key_from_seed(uint64_t seed) { return orc_mix64(seed + GAMMA); }
uint64_t orc_fork(uint64_t key, uint64_t tag) { return orc_mix64(key ^ orc_mix64(tag * GAMMA + 0x632BE59BD9B4E019ULL)); }

typedef struct {
    uint64_t key, ctr;
} rng_t;

static uint64_t next_u64(rng_t* r) {
    ++r->ctr;
    return orc_mix64(r->key + r->ctr * GAMMA);
}
static double uniform01(rng_t* r) { return (double)(next_u64(r) >> 11) * 0x1.0p-53; }
static double uniform(rng_t* r, double lo, double hi) { return lo + (hi - lo) * uniform01(r); }
static uint64_t uniform_int(rng_t* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)next_u64(r) * n) >> 64);
}
static double normal01(rng_t* r) {
    double u1 = uniform01(r);
    double u2 = uniform01(r);
    if (u1 <= 0.0) u1 = 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * PI * u2);
}

uint64_t orc_derive_episode_seed(uint64_t root, int episode) {  /* harness.hpp:25-27 */
    return orc_fork(orc_fork(orc_key_from_seed(root), 0xE915E915E915E915ULL), (uint64_t)episode);
}

int orc_policy_action(uint64_t seed, int step, int robot) {  /* harness.hpp:29-34, policy.hpp:448-449 */
    rng_t r = {orc_fork(orc_fork(orc_fork(orc_key_from_seed(seed), 0x9D0C7E5F00000001ULL), (uint64_t)step),
                        (uint64_t)robot),
               0};
    return (int)uniform_int(&r, 5);
}

void orc_rng_draws(uint64_t seed, uint64_t tag, int kind, uint64_t n, int count, double* out_f, uint64_t* out_u) {
    rng_t r = {orc_fork(orc_key_from_seed(seed), tag), 0};
    for (int i = 0; i < count; ++i) {
        if (kind == 0) out_u[i] = next_u64(&r);
        else if (kind == 1) out_f[i] = uniform01(&r);
        else if (kind == 2) out_f[i] = normal01(&r);
        else out_u[i] = uniform_int(&r, n);
    }
}

/* ---------------- core (core.hpp) ---------------- */

static double clampd(double v, double lo, double hi) {  /* core.hpp:144 */
    double m = v < lo ? lo : v;  /* std::max(v, lo) */
    return hi < m ? hi : m;      /* std::min(m, hi) */
}
static double dmin(double a, double b) { return b < a ? b : a; }  /* std::min */
static double dmax(double a, double b) { return a < b ? b : a; }  /* std::max */

static double wrap_angle(double t) {  /* core.hpp:102-108 */
    double r = remainder(t, 2.0 * PI);
    if (r <= -PI) r += 2.0 * PI;
    return r;
}

/* ---------------- QP (qp.hpp) ---------------- */

/* cholesky_solve (qp.hpp:65-89) */
static int cholesky_solve(double* M, double* x, int k) {
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j <= i; ++j) {
            double s = M[i * k + j];
            for (int p = 0; p < j; ++p) s -= M[i * k + p] * M[j * k + p];
            if (i == j) {
                if (s <= 1e-14) return 0;
                M[i * k + i] = sqrt(s);
            } else {
                M[i * k + j] = s / M[j * k + j];
            }
        }
    }
    for (int i = 0; i < k; ++i) {
        double s = x[i];
        for (int p = 0; p < i; ++p) s -= M[i * k + p] * x[p];
        x[i] = s / M[i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
        double s = x[i];
        for (int p = i + 1; p < k; ++p) s -= M[p * k + i] * x[p];
        x[i] = s / M[i * k + i];
    }
    return 1;
}

typedef struct {
    int n, total;
    double G[MAXROWS * MAXV];
    double h[MAXROWS];
} rowset_t;

/* fold_rows (qp.hpp:104-141) */
static void fold_rows(int n, int m, const double* A, const double* b, const double* lo, const double* hi,
                      rowset_t* rs) {
    rs->n = n;
    int t = 0;
    for (int r = 0; r < m; ++r) {
        double norm = 0.0;
        for (int i = 0; i < n; ++i) {
            double a = A[r * n + i];
            norm += a * a;
        }
        norm = sqrt(norm);
        if (norm < 1e-14) {
            for (int i = 0; i < n; ++i) rs->G[t * n + i] = 0.0;
            rs->h[t++] = b[r];
            continue;
        }
        for (int i = 0; i < n; ++i) rs->G[t * n + i] = A[r * n + i] / norm;
        rs->h[t++] = b[r] / norm;
    }
    for (int i = 0; i < n; ++i) {
        if (hi[i] < 1e30) {
            for (int q = 0; q < n; ++q) rs->G[t * n + q] = 0.0;
            rs->G[t * n + i] = 1.0;
            rs->h[t++] = hi[i];
        }
        if (lo[i] > -1e30) {
            for (int q = 0; q < n; ++q) rs->G[t * n + q] = 0.0;
            rs->G[t * n + i] = -1.0;
            rs->h[t++] = -lo[i];
        }
    }
    rs->total = t;
}

static double dot_u(const rowset_t* rs, int r, const double* u) {  /* qp.hpp:97-101 */
    double s = 0.0;
    for (int i = 0; i < rs->n; ++i) s += rs->G[r * rs->n + i] * u[i];
    return s;
}

/* solve_gram lambda (qp.hpp:199-221) */
static int solve_gram(const rowset_t* rs, const int* active, int k, const double* target, double* r) {
    double M[MAXV * MAXV];
    for (int a = 0; a < k; ++a) r[a] = 0.0;
    if (k == 0) return 1;
    for (int a = 0; a < k; ++a)
        for (int c = 0; c <= a; ++c) {
            double s = 0.0;
            for (int i = 0; i < rs->n; ++i) s += rs->G[active[a] * rs->n + i] * rs->G[active[c] * rs->n + i];
            M[a * k + c] = s;
            M[c * k + a] = s;
        }
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int i = 0; i < rs->n; ++i) s += rs->G[active[a] * rs->n + i] * target[i];
        r[a] = s;
    }
    return cholesky_solve(M, r, k);
}

static void erase_at(int* act, double* lam, int* k, int pos) {
    for (int q = pos; q < *k - 1; ++q) {
        act[q] = act[q + 1];
        lam[q] = lam[q + 1];
    }
    --*k;
}

static rowset_t g_rs; /* single-threaded test oracle: one scratch row set */

/* solve_qp (qp.hpp:183-357) without the KKT-residual diagnostic. */
int orc_solve_qp(int n, int m, const double* A, const double* b, const double* lo, const double* hi,
                 const double* u_nom, double tol, int max_iterations, double* u, int* iterations) {
    rowset_t* rs = &g_rs;
    for (int i = 0; i < n; ++i) u[i] = u_nom[i];
    fold_rows(n, m, A, b, lo, hi, rs);
    const int total = rs->total;
    if (max_iterations <= 0) max_iterations = 100 + 20 * total;
    int active[MAXROWS], k = 0;
    double lambda[MAXROWS];
    int iter = 0;
    for (; iter < max_iterations; ++iter) {
        int p = -1;
        double worst = tol;
        for (int r = 0; r < total; ++r) {
            int is_active = 0;
            for (int a = 0; a < k; ++a)
                if (active[a] == r) { is_active = 1; break; }
            if (is_active) continue;
            double v = dot_u(rs, r, u) - rs->h[r];
            if (v > worst) {
                worst = v;
                p = r;
            }
        }
        if (p < 0) break;
        {
            double gnorm = 0.0;
            for (int i = 0; i < n; ++i) {
                double g = rs->G[p * n + i];
                gnorm += g * g;
            }
            if (gnorm < 1e-14) {
                if (iterations) *iterations = iter;
                return 1;
            }
        }
        double np[MAXV];
        for (int i = 0; i < n; ++i) np[i] = rs->G[p * n + i];
        int added = 0;
        double lam_p = 0.0;
        for (int guard = 0; guard <= total && !added; ++guard) {
            double r[MAXROWS];
            if (!solve_gram(rs, active, k, np, r)) {
                int drop = 0;
                for (int i = 1; i < k; ++i)
                    if (lambda[i] < lambda[drop]) drop = i;
                erase_at(active, lambda, &k, drop);
                continue;
            }
            double z[MAXV];
            for (int i = 0; i < n; ++i) z[i] = np[i];
            for (int a = 0; a < k; ++a)
                for (int i = 0; i < n; ++i) z[i] -= r[a] * rs->G[active[a] * n + i];
            double z2 = 0.0;
            for (int i = 0; i < n; ++i) z2 += z[i] * z[i];
            double viol = dot_u(rs, p, u) - rs->h[p];
            if (viol <= tol) {
                if (lam_p > 0.0) {
                    active[k] = p;
                    lambda[k] = lam_p;
                    ++k;
                }
                added = 1;
                break;
            }
            double t1 = INFINITY;
            int blocker = -1;
            for (int a = 0; a < k; ++a) {
                if (r[a] > 1e-12) {
                    double t = lambda[a] / r[a];
                    if (t < t1) {
                        t1 = t;
                        blocker = a;
                    }
                }
            }
            if (z2 <= 1e-14) {
                if (blocker < 0) {
                    if (iterations) *iterations = iter;
                    return 1;
                }
                for (int a = 0; a < k; ++a) lambda[a] -= t1 * r[a];
                lam_p += t1;
                erase_at(active, lambda, &k, blocker);
                continue;
            }
            double t2 = viol / z2;
            double t = dmin(t1, t2);
            for (int i = 0; i < n; ++i) u[i] -= t * z[i];
            for (int a = 0; a < k; ++a) lambda[a] -= t * r[a];
            lam_p += t;
            if (t2 <= t1) {
                active[k] = p;
                lambda[k] = lam_p;
                ++k;
                added = 1;
            } else {
                erase_at(active, lambda, &k, blocker);
            }
        }
        if (!added) break;
    }
    if (iterations) *iterations = iter;
    return iter >= max_iterations ? 2 : 0;
}

/* ---------------- controller + barrier (controllers.hpp, barrier.hpp) ---------------- */

typedef struct {
    double v, w;
} cmd_t;

static cmd_t clamp_command(cmd_t c, const mrsim_cfg* p) {  /* core.hpp:146-148 */
    cmd_t o = {clampd(c.v, -p->v_max, p->v_max), clampd(c.w, -p->omega_max, p->omega_max)};
    return o;
}

/* position_waypoint_controller (controllers.hpp:86-92) via 34-55 */
static cmd_t position_controller(const mrsim_cfg* p, double x, double y, double th, double wx, double wy) {
    const double l = p->projection_distance;
    double px = x + cos(th) * l, py = y + sin(th) * l;
    double ux = p->k_position * (wx - px), uy = p->k_position * (wy - py);
    double nrm = hypot(ux, uy); /* clamp_si core.hpp:150-155 */
    if (!(nrm <= p->si_max_speed || nrm == 0.0)) {
        double s = p->si_max_speed / nrm;
        ux = ux * s;
        uy = uy * s;
    }
    const double c = cos(th), s = sin(th);
    cmd_t cmd = {c * ux + s * uy, (-s * ux + c * uy) / l};
    return clamp_command(cmd, p);
}

/* unicycle_pose_controller (controllers.hpp:68-82) */
static cmd_t pose_controller(const mrsim_cfg* p, double x, double y, double th, double gx, double gy, double gth) {
    const double dx = gx - x, dy = gy - y;
    const double rho = hypot(dx, dy);
    const double herr = wrap_angle(gth - th);
    cmd_t zero = {0.0, 0.0};
    if (rho < p->pose_position_tolerance && fabs(herr) < p->pose_heading_tolerance) return zero;
    const double alpha = wrap_angle(atan2(dy, dx) - th);
    const double beta = wrap_angle(gth - th - alpha);
    cmd_t cmd = {p->k_rho * rho, p->k_alpha * alpha + p->k_beta * beta};
    return clamp_command(cmd, p);
}

int orc_apply_barrier(const mrsim_cfg* p, int n, const double* poses, const double* nominal, int nobs,
                      const double* obstacles, const uint64_t* masks, double* commands, int* infeasible) {
    cmd_t out[MAXN];
    *infeasible = 0;
    for (int i = 0; i < n; ++i) {
        cmd_t c0 = {nominal[2 * i], nominal[2 * i + 1]};
        out[i] = clamp_command(c0, p);
    }
    if (!p->barrier_enabled || n == 0) goto done;
    {
        const double l = p->projection_distance;
        double qx[MAXN], qy[MAXN];
        for (int i = 0; i < n; ++i) {  /* projected_point */
            qx[i] = poses[3 * i] + cos(poses[3 * i + 2]) * l;
            qy[i] = poses[3 * i + 1] + sin(poses[3 * i + 2]) * l;
        }
        const double R = p->safety_radius + 2.0 * l + p->discrete_margin;   /* barrier.hpp:155 */
        const double bm = p->boundary_margin + l + p->discrete_margin;       /* barrier.hpp:156 */
        const double gamma = p->barrier_gain, r2 = R * R;
        const int nv = 2 * n;
        static double A[MAXROWS * MAXV], b[MAXROWS];
        int m = 0;
        /* build_barrier_constraints (barrier.hpp:57-121) */
        for (int i = 0; i < n; ++i)
            for (int j = i + 1; j < n; ++j) {
                double dx = qx[i] - qx[j], dy = qy[i] - qy[j];
                double dist2 = dx * dx + dy * dy;
                if (dist2 < 1e-18) return MRSIM_E_DOMAIN;
                double h = dist2 - r2;
                for (int q = 0; q < nv; ++q) A[m * nv + q] = 0.0;
                A[m * nv + 2 * i] = -2.0 * dx;
                A[m * nv + 2 * i + 1] = -2.0 * dy;
                A[m * nv + 2 * j] = 2.0 * dx;
                A[m * nv + 2 * j + 1] = 2.0 * dy;
                b[m++] = gamma * h * h * h;
            }
        const double xmin = -p->arena_half_width, xmax = p->arena_half_width;
        const double ymin = -p->arena_half_height, ymax = p->arena_half_height;
        for (int i = 0; i < n; ++i) {
            double wh[4] = {qx[i] - (xmin + bm), (xmax - bm) - qx[i], qy[i] - (ymin + bm), (ymax - bm) - qy[i]};
            double wc[4][2] = {{-1.0, 0.0}, {1.0, 0.0}, {0.0, -1.0}, {0.0, 1.0}};
            for (int w = 0; w < 4; ++w) {
                for (int q = 0; q < nv; ++q) A[m * nv + q] = 0.0;
                A[m * nv + 2 * i] = wc[w][0];
                A[m * nv + 2 * i + 1] = wc[w][1];
                b[m++] = gamma * wh[w] * wh[w] * wh[w];
            }
        }
        for (int i = 0; i < n; ++i)
            for (int o = 0; o < nobs; ++o) {
                if (masks && masks[o] != 0 && (masks[o] & (1ULL << i)) == 0) continue;
                double rad = obstacles[3 * o + 2];
                rad += l + p->discrete_margin;
                double dx = qx[i] - obstacles[3 * o], dy = qy[i] - obstacles[3 * o + 1];
                double h = (dx * dx + dy * dy) - rad * rad;
                for (int q = 0; q < nv; ++q) A[m * nv + q] = 0.0;
                A[m * nv + 2 * i] = -2.0 * dx;
                A[m * nv + 2 * i + 1] = -2.0 * dy;
                b[m++] = gamma * h * h * h;
            }
        double unom[MAXV], lo[MAXV], hi[MAXV], u[MAXV];
        for (int i = 0; i < n; ++i) {  /* uni_to_si (controllers.hpp:59-65) */
            double c = cos(poses[3 * i + 2]), s = sin(poses[3 * i + 2]);
            unom[2 * i] = c * out[i].v - l * s * out[i].w;
            unom[2 * i + 1] = s * out[i].v + l * c * out[i].w;
        }
        const double cap = p->v_max + l * p->omega_max + 0.1; /* barrier.hpp:173 */
        for (int q = 0; q < nv; ++q) {
            lo[q] = -cap;
            hi[q] = cap;
        }
        int it = 0;
        int st = orc_solve_qp(nv, m, A, b, lo, hi, unom, 1e-9, 0, u, &it);
        if (st == 1) {
            for (int i = 0; i < n; ++i) {
                out[i].v = 0.0;
                out[i].w = 0.0;
            }
            *infeasible = 1;
            goto done;
        }
        double scale = 1.0; /* map back (barrier.hpp:189-204) */
        cmd_t mapped[MAXN];
        for (int i = 0; i < n; ++i) {
            double c = cos(poses[3 * i + 2]), s = sin(poses[3 * i + 2]);
            mapped[i].v = c * u[2 * i] + s * u[2 * i + 1];
            mapped[i].w = (-s * u[2 * i] + c * u[2 * i + 1]) / l;
            if (fabs(mapped[i].v) > p->v_max) scale = dmin(scale, p->v_max / fabs(mapped[i].v));
            if (fabs(mapped[i].w) > p->omega_max) scale = dmin(scale, p->omega_max / fabs(mapped[i].w));
        }
        for (int i = 0; i < n; ++i) {
            out[i].v = mapped[i].v * scale;
            out[i].w = mapped[i].w * scale;
        }
    }
done:
    for (int i = 0; i < n; ++i) {
        commands[2 * i] = out[i].v;
        commands[2 * i + 1] = out[i].w;
    }
    return MRSIM_OK;
}

/* ---------------- scenarios (scenario.hpp, scenarios/*.hpp) ---------------- */

static int rect_contains(const double* r, double x, double y) {  /* core.hpp:35-37 */
    return x >= r[0] && x <= r[1] && y >= r[2] && y <= r[3];
}

static int requests_of(const mrsim_layout* y) {  /* rware.hpp:38-42 */
    int r = y->rware_request_size < y->rware_num_shelves ? y->rware_request_size : y->rware_num_shelves;
    return r > 0 ? r : 0;
}

int orc_obs_dim(const mrsim_cfg* c) {
    const int N = c->num_robots, base = 3 + 2 * (N - 1);
    const mrsim_layout* y = &c->layout;
    int d = 0;
    switch (c->task) {
        case MRSIM_TASK_NAVIGATION: d = 5; break;
        case MRSIM_TASK_PREDATOR_PREY: d = base + 2; break;
        case MRSIM_TASK_DISCOVERY: d = base + 2 * y->discovery_num_landmarks; break;
        case MRSIM_TASK_RWARE: d = base + 3 * y->rware_num_slots + requests_of(y) + 1; break;
        case MRSIM_TASK_FORAGING: d = base + 3 * y->foraging_num_resources; break;
        case MRSIM_TASK_MATERIAL_TRANSPORT: d = base + 3; break;
        case MRSIM_TASK_ARCTIC_TRANSPORT: {
            int drones = 0;
            for (int i = 0; i < N; ++i) drones += c->het[i][0] == 1.0;
            d = base + 1 + 9 * drones;
            break;
        }
        case MRSIM_TASK_WAREHOUSE: d = base + 1; break;
        case MRSIM_TASK_RANDOM_WAYPOINTS: d = 5; break;
    }
    if (c->het_obs_mode == MRSIM_HET_OBS_OWN) d += c->het_cols;
    else if (c->het_obs_mode == MRSIM_HET_OBS_FULL_TEAM) d += c->het_rows * c->het_cols;
    return d;
}

/* sample_poses (scenario.hpp:95-118) */
static int sample_poses(int n, double xmin, double xmax, double ymin, double ymax, double min_sep, rng_t* rng,
                        mrsim_env_state* s, int* bad) {
    for (int i = 0; i < n; ++i) {
        int placed = 0;
        for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
            double px = uniform(rng, xmin, xmax);
            double py = uniform(rng, ymin, ymax);
            double pt = PI * (1.0 - 2.0 * uniform01(rng));
            int ok = 1;
            for (int q = 0; q < i; ++q)
                if (hypot(px - s->x[q], py - s->y[q]) < min_sep) { ok = 0; break; }
            if (ok) {
                s->x[i] = px;
                s->y[i] = py;
                s->theta[i] = pt;
                placed = 1;
            }
        }
        if (!placed) {
            *bad = i;
            return 0;
        }
    }
    return 1;
}

static int arctic_tile_at(const mrsim_cfg* c, const mrsim_env_state* s, double x, double y) {
    /* arctic_transport.hpp:47-55 */
    const double xmin = -c->arena_half_width, xmax = c->arena_half_width;
    const double ymin = -c->arena_half_height, ymax = c->arena_half_height;
    double cw = (xmax - xmin) / s->cols, ch = (ymax - ymin) / s->rows;
    int cc = (int)((x - xmin) / cw), rr = (int)((y - ymin) / ch);
    cc = (int)clampd(cc, 0, s->cols - 1);
    rr = (int)clampd(rr, 0, s->rows - 1);
    return s->tiles[rr * s->cols + cc];
}

/* RandomWaypointsScenario::draw_target + heading draw (random_waypoints.hpp:24-27, 34-35, 62-63) */
static void rwp_draw(const mrsim_cfg* c, rng_t* rng, mrsim_env_state* s, int i) {
    const double m = c->layout.rwp_waypoint_margin;
    const double hw = c->arena_half_width, hh = c->arena_half_height;
    s->targets[i][0] = uniform(rng, -hw + m, hw - m);
    s->targets[i][1] = uniform(rng, -hh + m, hh - m);
    s->target_headings[i] = PI * (1.0 - 2.0 * uniform01(rng));
}

int orc_reset_env(const mrsim_cfg* c, uint64_t seed, mrsim_env_state* s, char* err, int errlen) {
    const mrsim_layout* y = &c->layout;
    const int N = c->num_robots;
    memset(s, 0, sizeof *s);
    s->num_robots = N;
    s->rng_key = orc_key_from_seed(seed); /* batch.hpp:155 */
    s->seed = seed;
    s->episode = -1;
    s->min_pairwise_distance = INFINITY;
    rng_t rng = {orc_fork(s->rng_key, 0), 0}; /* reset_stream (scenario.hpp:87-88) */
    const double hw = c->arena_half_width, hh = c->arena_half_height;
    const double sm = y->spawn_margin, sep = c->safety_radius + y->spawn_separation_slack;
    int bad = 0, ok;
    if (c->task == MRSIM_TASK_ARCTIC_TRANSPORT)
        ok = sample_poses(N, y->arctic_spawn_zone[0], y->arctic_spawn_zone[1], y->arctic_spawn_zone[2],
                          y->arctic_spawn_zone[3], sep, &rng, s, &bad);
    else
        ok = sample_poses(N, -hw + sm, hw - sm, -hh + sm, hh - sm, sep, &rng, s, &bad);
    if (!ok) {
        char buf[128];
        snprintf(buf, sizeof buf, "sample_poses: could not place robot %d after 1000 attempts", bad);
        return fail(err, errlen, MRSIM_E_RUNTIME, buf);
    }
    switch (c->task) {
        case MRSIM_TASK_NAVIGATION: { /* navigation.hpp:55-75 */
            const double gm = y->navigation_goal_margin;
            for (int i = 0; i < N; ++i) {
                int placed = 0;
                for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
                    double gx = uniform(&rng, -hw + gm, hw - gm);
                    double gy = uniform(&rng, -hh + gm, hh - gm);
                    int good = 1;
                    for (int q = 0; q < i; ++q)
                        if (hypot(gx - s->goals[q][0], gy - s->goals[q][1]) < y->navigation_goal_separation) {
                            good = 0;
                            break;
                        }
                    if (good) {
                        s->goals[i][0] = gx;
                        s->goals[i][1] = gy;
                        placed = 1;
                    }
                }
                if (!placed) return fail(err, errlen, MRSIM_E_RUNTIME, "navigation: could not place goals");
            }
            break;
        }
        case MRSIM_TASK_PREDATOR_PREY: { /* predator_prey.hpp:48-66 */
            int placed = 0;
            for (int attempt = 0; attempt < 1000 && !placed; ++attempt) {
                double px = uniform(&rng, -hw + sm, hw - sm);
                double py = uniform(&rng, -hh + sm, hh - sm);
                int good = 1;
                for (int q = 0; q < N; ++q)
                    if (hypot(px - s->x[q], py - s->y[q]) < y->pp_prey_spawn_clearance) { good = 0; break; }
                if (good) {
                    s->prey[0] = px;
                    s->prey[1] = py;
                    placed = 1;
                }
            }
            if (!placed) return fail(err, errlen, MRSIM_E_RUNTIME, "predator_prey: could not place prey");
            break;
        }
        case MRSIM_TASK_DISCOVERY: { /* discovery.hpp:27-38 */
            const double lm = y->discovery_landmark_margin;
            s->num_landmarks = y->discovery_num_landmarks;
            for (int k = 0; k < s->num_landmarks; ++k) {
                s->landmarks[k][0] = uniform(&rng, -hw + lm, hw - lm);
                s->landmarks[k][1] = uniform(&rng, -hh + lm, hh - lm);
            }
            break;
        }
        case MRSIM_TASK_RWARE: { /* rware.hpp:25-44 */
            const int shelves = y->rware_num_shelves;
            s->num_slots = y->rware_num_slots;
            for (int q = 0; q < s->num_slots; ++q) s->slot_shelf[q] = q < shelves ? q + 1 : 0;
            int pool[MRSIM_MAX_SLOTS], np = 0;
            for (int i = 1; i <= shelves; ++i) pool[np++] = i;
            for (int k = 0; k < y->rware_request_size && np > 0; ++k) {
                int idx = (int)uniform_int(&rng, (uint64_t)np);
                s->requests[s->num_requests++] = pool[idx];
                for (int q = idx; q < np - 1; ++q) pool[q] = pool[q + 1];
                --np;
            }
            break;
        }
        case MRSIM_TASK_FORAGING: { /* foraging.hpp:27-49 */
            double l0 = -INFINITY, l1 = -INFINITY;
            for (int i = 0; i < c->het_rows; ++i) {
                double v = c->het[i][0];
                if (v > l0) { l1 = l0; l0 = v; } else if (v > l1) { l1 = v; }
            }
            double top2 = l0 + (c->het_rows > 1 ? l1 : 0.0);
            int max_level = (int)top2;
            if (max_level < 1) max_level = 1;
            const double rm = y->foraging_resource_margin;
            s->num_resources = y->foraging_num_resources;
            for (int r = 0; r < s->num_resources; ++r) {
                s->resources[r][0] = uniform(&rng, -hw + rm, hw - rm);
                s->resources[r][1] = uniform(&rng, -hh + rm, hh - rm);
                s->levels[r] = 1 + (int)uniform_int(&rng, (uint64_t)max_level);
            }
            break;
        }
        case MRSIM_TASK_MATERIAL_TRANSPORT: { /* material_transport.hpp:28-40 */
            double a = y->mt_circle_mean + sqrt(y->mt_circle_variance) * normal01(&rng);
            s->circle_remaining = dmax(0.0, round(a));
            double b = y->mt_rect_mean + sqrt(y->mt_rect_variance) * normal01(&rng);
            s->rect_remaining = dmax(0.0, round(b));
            s->total_initial = s->circle_remaining + s->rect_remaining;
            break;
        }
        case MRSIM_TASK_ARCTIC_TRANSPORT: { /* arctic_transport.hpp:30-45 */
            s->cols = y->arctic_grid_cols;
            s->rows = y->arctic_grid_rows;
            memcpy(s->goal_zone, y->arctic_goal_zone, sizeof s->goal_zone);
            for (int r = 0; r < s->rows; ++r)
                for (int cc = y->arctic_ground_cols_left; cc < s->cols - y->arctic_ground_cols_right; ++cc)
                    s->tiles[r * s->cols + cc] = uniform_int(&rng, 2) == 0 ? 1 : 2;
            break;
        }
        case MRSIM_TASK_RANDOM_WAYPOINTS: /* random_waypoints.hpp:29-37 */
            for (int i = 0; i < N; ++i) {
                rwp_draw(c, &rng, s, i);
            }
            break;
        default:
            break;
    }
    return MRSIM_OK;
}

/* Scenario::transition (scenarios/*.hpp) */
static double transition(const mrsim_cfg* c, mrsim_env_state* s, rng_t* rng) {
    const int N = c->num_robots;
    const mrsim_layout* y = &c->layout;
    switch (c->task) {
        case MRSIM_TASK_RANDOM_WAYPOINTS: { /* random_waypoints.hpp:52-66 (sequential over robots) */
            for (int i = 0; i < N; ++i) {
                double cx = s->x[i], cy = s->y[i];
                if (c->controller == MRSIM_CONTROLLER_UNICYCLE_POSITION) { /* projected_point */
                    cx = s->x[i] + cos(s->theta[i]) * c->projection_distance;
                    cy = s->y[i] + sin(s->theta[i]) * c->projection_distance;
                }
                if (hypot(cx - s->targets[i][0], cy - s->targets[i][1]) <= y->rwp_arrival_tolerance)
                    rwp_draw(c, rng, s, i);
            }
            return 0.0;
        }
        case MRSIM_TASK_NAVIGATION: { /* navigation.hpp:45-51 */
            double total = 0.0;
            for (int i = 0; i < N; ++i) total += hypot(s->x[i] - s->goals[i][0], s->y[i] - s->goals[i][1]);
            return c->coef[MRSIM_COEF_DIST] * total;
        }
        case MRSIM_TASK_PREDATOR_PREY: { /* predator_prey.hpp:15-34, 177-199 */
            double robot_step = 0.0;
            for (int i = 0; i < N; ++i) robot_step = dmax(robot_step, c->step_sizes[i]);
            double step = y->pp_prey_agility * robot_step;
            double bx = s->prey[0], by = s->prey[1], best = -INFINITY;
            for (int k = 0; k < 9; ++k) {
                double cx = s->prey[0], cy = s->prey[1];
                if (k > 0) {
                    double ang = (k - 1) * (PI / 4.0);
                    cx = s->prey[0] + cos(ang) * step;
                    cy = s->prey[1] + sin(ang) * step;
                }
                if (!(cx >= -c->arena_half_width && cx <= c->arena_half_width && cy >= -c->arena_half_height &&
                      cy <= c->arena_half_height))
                    continue;
                double nearest = INFINITY;
                for (int i = 0; i < N; ++i) nearest = dmin(nearest, hypot(cx - s->x[i], cy - s->y[i]));
                if (nearest > best) {
                    best = nearest;
                    bx = cx;
                    by = cy;
                }
            }
            s->prey[0] = bx;
            s->prey[1] = by;
            int tagged = 0;
            for (int i = 0; i < N; ++i) tagged = tagged || hypot(s->x[i] - bx, s->y[i] - by) <= y->pp_tag_radius;
            if (tagged) {
                s->scenario_metric += 1.0;
                s->flash_timer = y->pp_flash_steps;
            } else if (s->flash_timer > 0) {
                --s->flash_timer;
            }
            return tagged ? c->coef[MRSIM_COEF_TAG] : 0.0;
        }
        case MRSIM_TASK_DISCOVERY: { /* discovery.hpp:40-69 */
            int ns = 0, nt = 0;
            for (int k = 0; k < s->num_landmarks; ++k) {
                if (s->tagged[k]) continue;
                int sh = 0, th = 0;
                for (int i = 0; i < N; ++i) {
                    double d = hypot(s->x[i] - s->landmarks[k][0], s->y[i] - s->landmarks[k][1]);
                    if (c->het[i][0] > 0.0 && d <= c->het[i][0]) sh = 1;
                    if (c->het[i][1] > 0.0 && d <= c->het[i][1]) th = 1;
                }
                if (sh && !s->sensed[k]) {
                    s->sensed[k] = 1;
                    ++ns;
                }
                if (th) {
                    s->tagged[k] = 1;
                    ++nt;
                }
            }
            int all = 1;
            for (int k = 0; k < s->num_landmarks; ++k) all = all && s->tagged[k];
            s->scenario_metric += nt;
            return c->coef[MRSIM_COEF_SENSE] * ns + c->coef[MRSIM_COEF_TAG] * nt +
                   c->coef[MRSIM_COEF_STEP] * (all ? 0.0 : 1.0);
        }
        case MRSIM_TASK_RWARE: { /* rware.hpp:70-107 */
            double reward = 0.0;
            const int R = s->num_requests;
            for (int i = 0; i < N; ++i) {
                double px = s->x[i], py = s->y[i];
                if (s->carried[i] != 0 && rect_contains(y->rware_dropoff_zone, px, py)) {
                    int it = -1;
                    for (int q = 0; q < R; ++q)
                        if (s->requests[q] == s->carried[i]) { it = q; break; }
                    if (it >= 0) {
                        reward += c->coef[MRSIM_COEF_DROPOFF];
                        s->scenario_metric += 1.0;
                        int cand[MRSIM_MAX_SLOTS], nc = 0;
                        for (int id = 1; id <= y->rware_num_shelves; ++id) {
                            int req = 0;
                            for (int q = 0; q < R; ++q) req = req || s->requests[q] == id;
                            if (!req) cand[nc++] = id;
                        }
                        if (nc > 0) s->requests[it] = cand[uniform_int(rng, (uint64_t)nc)];
                    }
                    continue;
                }
                int slot = -1;
                for (int q = 0; q < s->num_slots; ++q)
                    if (fabs(px - y->rware_slots[2 * q]) <= y->rware_slot_half &&
                        fabs(py - y->rware_slots[2 * q + 1]) <= y->rware_slot_half) {
                        slot = q;
                        break;
                    }
                if (slot < 0) continue;
                if (s->carried[i] == 0 && s->slot_shelf[slot] != 0) {
                    s->carried[i] = s->slot_shelf[slot];
                    s->slot_shelf[slot] = 0;
                } else if (s->carried[i] != 0 && s->slot_shelf[slot] == 0) {
                    s->slot_shelf[slot] = s->carried[i];
                    s->carried[i] = 0;
                }
            }
            return reward;
        }
        case MRSIM_TASK_FORAGING: { /* foraging.hpp:51-70 */
            double reward = 0.0;
            for (int r = 0; r < s->num_resources; ++r) {
                if (s->foraged[r]) continue;
                double sum = 0.0;
                for (int i = 0; i < N; ++i)
                    if (hypot(s->x[i] - s->resources[r][0], s->y[i] - s->resources[r][1]) <= y->foraging_radius)
                        sum += c->het[i][0];
                if (sum >= s->levels[r]) {
                    s->foraged[r] = 1;
                    reward += c->coef[MRSIM_COEF_FORAGE] * s->levels[r];
                    s->scenario_metric += 1.0;
                }
            }
            return reward;
        }
        case MRSIM_TASK_MATERIAL_TRANSPORT: { /* material_transport.hpp:42-74 */
            double loaded = 0.0, dropped = 0.0;
            for (int i = 0; i < N; ++i) {
                double px = s->x[i], py = s->y[i], cap = c->het[i][1];
                if (s->loads[i] > 0.0 && rect_contains(y->mt_dropoff_zone, px, py)) {
                    dropped += s->loads[i];
                    s->delivered += s->loads[i];
                    s->loads[i] = 0.0;
                } else if (s->loads[i] == 0.0) {
                    if (hypot(y->mt_circle_zone[0] - px, y->mt_circle_zone[1] - py) <= y->mt_circle_zone[2] &&
                        s->circle_remaining > 0.0) {
                        double take = dmin(cap, s->circle_remaining);
                        s->circle_remaining -= take;
                        s->loads[i] = take;
                        loaded += take;
                    } else if (rect_contains(y->mt_rect_zone, px, py) && s->rect_remaining > 0.0) {
                        double take = dmin(cap, s->rect_remaining);
                        s->rect_remaining -= take;
                        s->loads[i] = take;
                        loaded += take;
                    }
                }
            }
            s->scenario_metric = s->circle_remaining + s->rect_remaining;
            int empty = s->circle_remaining == 0.0 && s->rect_remaining == 0.0;
            return c->coef[MRSIM_COEF_LOAD] * loaded + c->coef[MRSIM_COEF_DROPOFF] * dropped +
                   c->coef[MRSIM_COEF_STEP] * (empty ? 0.0 : 1.0);
        }
        case MRSIM_TASK_ARCTIC_TRANSPORT: { /* arctic_transport.hpp:75-86 */
            double sum = 0.0;
            int all = 1;
            for (int i = 0; i < N; ++i) {
                if (c->het[i][0] == 1.0) continue;
                double px = s->x[i], py = s->y[i];
                double dx = dmax(dmax(s->goal_zone[0] - px, 0.0), px - s->goal_zone[1]);
                double dy = dmax(dmax(s->goal_zone[2] - py, 0.0), py - s->goal_zone[3]);
                sum += hypot(dx, dy);
                all = all && rect_contains(s->goal_zone, px, py);
            }
            return c->coef[MRSIM_COEF_DIST] * sum + c->coef[MRSIM_COEF_STEP] * (all ? 0.0 : 1.0);
        }
        case MRSIM_TASK_WAREHOUSE: { /* warehouse.hpp:36-54 */
            double reward = 0.0;
            for (int i = 0; i < N; ++i) {
                double px = s->x[i], py = s->y[i];
                int green = c->het[i][0] == 1.0;
                const double* pick = green ? y->warehouse_green_right : y->warehouse_red_right;
                const double* del = green ? y->warehouse_green_left : y->warehouse_red_left;
                if (!s->loaded[i] && rect_contains(pick, px, py)) {
                    s->loaded[i] = 1;
                    reward += c->coef[MRSIM_COEF_LOAD];
                } else if (s->loaded[i] && rect_contains(del, px, py)) {
                    s->loaded[i] = 0;
                    reward += c->coef[MRSIM_COEF_DELIVERY];
                    s->scenario_metric += 1.0;
                }
            }
            return reward;
        }
    }
    return 0.0;
}

static void finalize(const mrsim_cfg* c, mrsim_env_state* s) {
    if (c->task == MRSIM_TASK_NAVIGATION) { /* navigation.hpp:53-61 */
        int all = 1;
        for (int i = 0; i < c->num_robots; ++i)
            all = all && hypot(s->x[i] - s->goals[i][0], s->y[i] - s->goals[i][1]) <= c->layout.navigation_on_goal_radius;
        s->success = all;
        s->scenario_metric = all ? 1.0 : 0.0;
    } else if (c->task == MRSIM_TASK_ARCTIC_TRANSPORT) { /* arctic_transport.hpp:88-97 */
        int all = 1;
        for (int i = 0; i < c->num_robots; ++i) {
            if (c->het[i][0] == 1.0) continue;
            all = all && rect_contains(s->goal_zone, s->x[i], s->y[i]);
        }
        s->success = all;
        s->scenario_metric = all ? 1.0 : 0.0;
    }
}

int orc_observe(const mrsim_cfg* c, const mrsim_env_state* s, double* obs) {
    const int N = c->num_robots, D = orc_obs_dim(c);
    const mrsim_layout* y = &c->layout;
    for (int r = 0; r < N; ++r) {
        double* o = obs + r * D;
        int q = 0;
        if (c->task == MRSIM_TASK_RANDOM_WAYPOINTS) { /* random_waypoints.hpp:70-76 */
            o[q++] = s->x[r];
            o[q++] = s->y[r];
            o[q++] = s->theta[r];
            o[q++] = s->targets[r][0];
            o[q++] = s->targets[r][1];
        } else if (c->task == MRSIM_TASK_NAVIGATION) { /* navigation.hpp:64-70 */
            o[q++] = s->x[r];
            o[q++] = s->y[r];
            o[q++] = s->theta[r];
            o[q++] = s->goals[r][0] - s->x[r];
            o[q++] = s->goals[r][1] - s->y[r];
        } else {
            o[q++] = s->x[r]; /* base_observation (scenario.hpp:200-210) */
            o[q++] = s->y[r];
            o[q++] = s->theta[r];
            for (int j = 0; j < N; ++j) {
                if (j == r) continue;
                o[q++] = s->x[j];
                o[q++] = s->y[j];
            }
            switch (c->task) {
                case MRSIM_TASK_PREDATOR_PREY:
                    o[q++] = s->prey[0];
                    o[q++] = s->prey[1];
                    break;
                case MRSIM_TASK_DISCOVERY:
                    for (int k = 0; k < s->num_landmarks; ++k) {
                        int vis = s->sensed[k] && !s->tagged[k];
                        o[q++] = vis ? s->landmarks[k][0] : y->discovery_sentinel[0];
                        o[q++] = vis ? s->landmarks[k][1] : y->discovery_sentinel[1];
                    }
                    break;
                case MRSIM_TASK_RWARE:
                    for (int k = 0; k < s->num_slots; ++k) {
                        o[q++] = y->rware_slots[2 * k];
                        o[q++] = y->rware_slots[2 * k + 1];
                        o[q++] = s->slot_shelf[k];
                    }
                    for (int k = 0; k < s->num_requests; ++k) o[q++] = s->requests[k];
                    o[q++] = s->carried[r];
                    break;
                case MRSIM_TASK_FORAGING:
                    for (int k = 0; k < s->num_resources; ++k) {
                        int live = !s->foraged[k];
                        o[q++] = live ? s->resources[k][0] : y->discovery_sentinel[0];
                        o[q++] = live ? s->resources[k][1] : y->discovery_sentinel[1];
                        o[q++] = live ? (double)s->levels[k] : 0.0;
                    }
                    break;
                case MRSIM_TASK_MATERIAL_TRANSPORT:
                    o[q++] = s->loads[r];
                    o[q++] = s->circle_remaining;
                    o[q++] = s->rect_remaining;
                    break;
                case MRSIM_TASK_ARCTIC_TRANSPORT: {
                    o[q++] = arctic_tile_at(c, s, s->x[r], s->y[r]);
                    const double xmin = -c->arena_half_width, xmax = c->arena_half_width;
                    const double ymin = -c->arena_half_height, ymax = c->arena_half_height;
                    double cw = (xmax - xmin) / s->cols, ch = (ymax - ymin) / s->rows;
                    for (int d = 0; d < N; ++d) {
                        if (c->het[d][0] != 1.0) continue;
                        int c0 = (int)clampd((s->x[d] - xmin) / cw, 0.0, s->cols - 1.0);
                        int r0 = (int)clampd((s->y[d] - ymin) / ch, 0.0, s->rows - 1.0);
                        for (int dr = -1; dr <= 1; ++dr)
                            for (int dc = -1; dc <= 1; ++dc) {
                                int rr = r0 + dr, cc = c0 + dc;
                                int in = rr >= 0 && rr < s->rows && cc >= 0 && cc < s->cols;
                                o[q++] = in ? s->tiles[rr * s->cols + cc] : 0;
                            }
                    }
                    break;
                }
                case MRSIM_TASK_WAREHOUSE:
                    o[q++] = s->loaded[r] ? 1.0 : 0.0;
                    break;
            }
        }
        if (c->het_obs_mode == MRSIM_HET_OBS_OWN) /* het_augment (framework.hpp:61-76) */
            for (int k = 0; k < c->het_cols; ++k) o[q++] = c->het[r][k];
        else if (c->het_obs_mode == MRSIM_HET_OBS_FULL_TEAM)
            for (int i = 0; i < c->het_rows; ++i)
                for (int k = 0; k < c->het_cols; ++k) o[q++] = c->het[i][k];
    }
    return MRSIM_OK;
}

int orc_step_env(const mrsim_cfg* c, mrsim_env_state* s, const int32_t* actions, double* obs, double* reward,
                 int* done, char* err, int errlen) {
    const int N = c->num_robots;
    const mrsim_layout* y = &c->layout;
    for (int r = 0; r < N; ++r)
        if (actions[r] < 0 || actions[r] > 4) {
            char buf[128];
            snprintf(buf, sizeof buf, "step_batch: invalid action %d for robot %d", actions[r], r);
            return fail(err, errlen, MRSIM_E_INVALID_ARGUMENT, buf);
        }
    rng_t rng = {orc_fork(s->rng_key, 1 + (uint64_t)s->step_index), 0}; /* step_stream (scenario.hpp:89-91) */
    double wx[MAXN], wy[MAXN];
    for (int i = 0; i < N; ++i) { /* waypoints (scenario.hpp:156-165) + action_to_waypoint (framework.hpp:96-108) */
        double size = c->step_sizes[i];
        if (c->task == MRSIM_TASK_ARCTIC_TRANSPORT) { /* arctic_transport.hpp:58-73 */
            size = y->arctic_normal_step;
            if (c->het[i][0] != 1.0) {
                int tile = arctic_tile_at(c, s, s->x[i], s->y[i]);
                if (tile != 0) {
                    int match = (c->het[i][1] == 1.0 && tile == 2) || (c->het[i][2] == 1.0 && tile == 1);
                    size = match ? y->arctic_fast_step : y->arctic_slow_step;
                }
            }
        }
        static const double DX[5] = {0.0, 0.0, 0.0, -1.0, 1.0}, DY[5] = {0.0, 1.0, -1.0, 0.0, 0.0};
        double px = s->x[i] + DX[actions[i]] * size;
        double py = s->y[i] + DY[actions[i]] * size;
        if (c->action_noise_scale > 0.0 && c->task != MRSIM_TASK_RANDOM_WAYPOINTS) {
            double half = c->action_noise_scale * size;
            px += uniform(&rng, -half, half);
            py += uniform(&rng, -half, half);
        }
        wx[i] = clampd(px, -c->arena_half_width, c->arena_half_width);
        wy[i] = clampd(py, -c->arena_half_height, c->arena_half_height);
        if (c->task == MRSIM_TASK_RANDOM_WAYPOINTS) { /* actions ignored (random_waypoints.hpp:40-44) */
            wx[i] = s->targets[i][0];
            wy[i] = s->targets[i][1];
        }
    }
    double wth[MAXN]; /* waypoint_headings for the pose controller (batch.hpp:169-171) */
    if (c->controller == MRSIM_CONTROLLER_UNICYCLE_POSE)
        for (int i = 0; i < N; ++i) {
            if (c->task == MRSIM_TASK_RANDOM_WAYPOINTS) { /* random_waypoints.hpp:46-50 */
                wth[i] = s->target_headings[i];
            } else { /* scenario.hpp:168-177 */
                double dx = wx[i] - s->x[i], dy = wy[i] - s->y[i];
                wth[i] = hypot(dx, dy) > 1e-12 ? atan2(dy, dx) : s->theta[i];
            }
        }
    /* add_obstacles (rware.hpp:54-68) */
    double obst[MRSIM_MAX_SLOTS * 3];
    uint64_t masks[MRSIM_MAX_SLOTS];
    int nobs = 0;
    if (c->task == MRSIM_TASK_RWARE) {
        uint64_t carriers = 0;
        for (int i = 0; i < N; ++i)
            if (s->carried[i] != 0) carriers |= 1ULL << i;
        if (carriers != 0)
            for (int q = 0; q < s->num_slots; ++q) {
                if (s->slot_shelf[q] == 0) continue;
                obst[3 * nobs] = y->rware_slots[2 * q];
                obst[3 * nobs + 1] = y->rware_slots[2 * q + 1];
                obst[3 * nobs + 2] = y->rware_shelf_radius;
                masks[nobs++] = carriers;
            }
    }
    int collision = 0;
    for (int tick = 0; tick < c->sub_steps; ++tick) { /* batch.hpp:181-210 */
        double poses[3 * MAXN], nom[2 * MAXN], cmd[2 * MAXN];
        for (int i = 0; i < N; ++i) {
            poses[3 * i] = s->x[i];
            poses[3 * i + 1] = s->y[i];
            poses[3 * i + 2] = s->theta[i];
            if (c->controller == MRSIM_CONTROLLER_UNICYCLE_POSE) {
                cmd_t k = pose_controller(c, s->x[i], s->y[i], s->theta[i], wx[i], wy[i], wth[i]);
                nom[2 * i] = k.v;
                nom[2 * i + 1] = k.w;
            } else if (wx[i] == s->x[i] && wy[i] == s->y[i]) {
                nom[2 * i] = 0.0;
                nom[2 * i + 1] = 0.0;
            } else {
                cmd_t k = position_controller(c, s->x[i], s->y[i], s->theta[i], wx[i], wy[i]);
                nom[2 * i] = k.v;
                nom[2 * i + 1] = k.w;
            }
        }
        int inf = 0;
        mrsim_cfg cb = *c;
        int rc = orc_apply_barrier(&cb, N, poses, nom, nobs, obst, masks, cmd, &inf);
        if (rc) return fail(err, errlen, rc, "build_barrier_constraints: coincident robot positions");
        if (inf) s->qp_infeasible += 1;
        for (int i = 0; i < N; ++i) { /* step_unicycle (core.hpp:112-118) + arena clamp */
            double th = s->theta[i];
            double nx = s->x[i] + cmd[2 * i] * cos(th) * c->dt;
            double ny = s->y[i] + cmd[2 * i] * sin(th) * c->dt;
            double nt = th + cmd[2 * i + 1] * c->dt;
            if (!isfinite(nt)) return fail(err, errlen, MRSIM_E_DOMAIN, "wrap_angle: non-finite input");
            s->theta[i] = wrap_angle(nt);
            s->x[i] = clampd(nx, -c->arena_half_width, c->arena_half_width);
            s->y[i] = clampd(ny, -c->arena_half_height, c->arena_half_height);
        }
        if (N > 1) { /* min_pairwise_distance (core.hpp:136-142) */
            double best = INFINITY;
            for (int i = 0; i < N; ++i)
                for (int j = i + 1; j < N; ++j) best = dmin(best, hypot(s->x[i] - s->x[j], s->y[i] - s->y[j]));
            s->min_pairwise_distance = dmin(s->min_pairwise_distance, best);
            collision = collision || best < c->collision_radius;
        }
    }
    double rew = transition(c, s, &rng); /* batch.hpp:212-223 */
    if (collision) {
        s->collisions += 1;
        rew += c->coef[MRSIM_COEF_VIOLATION];
    }
    s->step_index += 1;
    int d = s->step_index >= c->max_steps;
    if (d) finalize(c, s);
    s->episode_return += rew;
    if (reward) *reward = rew;
    if (done) *done = d;
    if (obs) orc_observe(c, s, obs);
    return MRSIM_OK;
}

/* ---------------- feedforward policy (policy.hpp:95-116, 445-480) ---------------- */

int orc_policy_act(const mrsim_cfg* c, const mrsim_env_state* s, int robot, int num_layers, const int32_t* dims,
                   const int32_t* acts, const double* weights, int greedy) {
    double obs[MAXN * 128], buf[2][256];
    const int D = orc_obs_dim(c);
    orc_observe(c, s, obs); /* assemble_observations (batch.hpp:143-151) */
    for (int i = 0; i < D; ++i) buf[0][i] = obs[robot * D + i];
    int cur = 0;
    const double* w = weights;
    for (int l = 0; l < num_layers; ++l) { /* FeedforwardWeights::forward */
        const int in = dims[2 * l], out = dims[2 * l + 1];
        const double* b = w + in * out;
        for (int o = 0; o < out; ++o) {
            double acc = b[o];
            for (int i = 0; i < in; ++i) acc += w[o * in + i] * buf[cur][i];
            if (acts[l] == MRSIM_ACT_RELU) acc = acc > 0 ? acc : 0;
            else if (acts[l] == MRSIM_ACT_TANH) acc = tanh(acc);
            buf[cur ^ 1][o] = acc;
        }
        w = b + out;
        cur ^= 1;
    }
    const double* lg = buf[cur];
    if (greedy) {
        int best = 0;
        for (int a = 1; a < 5; ++a)
            if (lg[a] > lg[best]) best = a;
        return best;
    }
    double mx = lg[0], p[5], z = 0.0;
    for (int a = 0; a < 5; ++a) mx = dmax(mx, lg[a]);
    for (int a = 0; a < 5; ++a) {
        p[a] = exp(lg[a] - mx);
        z += p[a];
    }
    /* policy_stream(seed, step, robot) (harness.hpp:29-34) */
    rng_t rng = {orc_fork(orc_fork(orc_fork(orc_key_from_seed(s->seed), 0x9D0C7E5F00000001ULL), (uint64_t)s->step_index),
                          (uint64_t)robot), 0};
    double u = uniform01(&rng) * z;
    for (int a = 0; a < 5; ++a) {
        u -= p[a];
        if (u <= 0.0) return a;
    }
    return 4;
}
