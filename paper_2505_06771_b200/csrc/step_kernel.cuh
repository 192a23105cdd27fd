// step_kernel.cuh — the fused per-step kernel: one group of L lanes per
// environment runs step_env (batch.hpp:165-224) end to end with the env's
// state in registers and shared memory, touching HBM once per step:
//
//   actions -> waypoints (framework.hpp:96-108, scenario.hpp:150-165)
//   sub_steps x [ hold rule / position controller (controllers.hpp:34-92)
//                 -> CBF rows + active-set QP + map back (barrier.hpp:57-205, qp.hpp)
//                 -> unicycle Euler + wrap + arena clamp (core.hpp:102-118, batch.hpp:199-203)
//                 -> min pairwise distance / collision flag (batch.hpp:204-209) ]
//   -> transition / violation / step_index / done / finalize (batch.hpp:212-220)
//   -> observations (batch.hpp:143-151, 221) -> optional in-kernel auto-reset.
//
// Lane v of the group owns QP variable v = 2*robot + axis; both lanes of a
// robot carry that robot's pose redundantly (no divergence, no extra
// traffic). Pair rows are spread over all lanes; reductions are shuffles.
#pragma once

#include "mrsim_device.cuh"
#include "qp_group.cuh"
#include "tasks.cuh"

namespace mrsim_dev {

// SoA batch state in HBM (one copy; the context ping-pongs two copies so a
// step is transactional: step_batch is pure, batch.hpp:267).
template <class Real>
struct DevState {
    Real *px, *py, *pt;                        // [B*N], env-major
    int32_t* step_index;                       // [B]
    uint64_t *key, *seed, *pkey;               // base rng key, episode seed, policy key prefix
    int64_t* episode;                          // [B]
    int32_t *collisions, *qp_inf, *success;    // [B]
    Real *metric, *min_dist, *ep_return;       // [B]
    Real* tf;                                  // [nf][B]
    int32_t* ti;                               // [ni][B]
};

// Per-env accumulators over completed episodes (single buffer).
struct EnvStats {
    int32_t* episodes;
    double *ret, *ret_sq, *metric, *success, *min_dist;
    int64_t *collisions, *qp_inf;
};

// Derived constants: SimParams, gains, BarrierConfig with the projection
// inflation of apply_barrier (barrier.hpp:151-157, 173).
template <class Real>
struct PhysConsts {
    Real dt, v_max, w_max, si_max, hw, hh, coll_r, k_pos, l, gamma, r_eff2, cap, obs_r_eff2, tol;
    Real wall_xmin, wall_xmax, wall_ymin, wall_ymax;
};

template <class Real>
struct StepParams {
    mrsim_cfg c;
    DevState<Real> in, out;
    EnvStats st;
    const int8_t* actions;  // [B][N] or nullptr (on-device random policy)
    float* obs;             // [B][N][D] or nullptr
    float* reward;          // [B] or nullptr
    double* reward64;       // [B] or nullptr (host-API path: the reference's double team reward)
    uint8_t* done;          // [B] or nullptr
    float* next_obs;        // [B][N][D] or nullptr
    unsigned long long* err;
    long long* err_serial;
    long long serial;
    long long B;
    int N, n, P, D, bdim, nf, ni;
    int auto_reset;
    uint64_t root_seed;
    long long episode_stride;
    int smem_bytes_per_group;
    PhysConsts<Real> k;
};

// Lexicographic pair index -> (i, j), i < j (barrier.hpp:69-83 order).
__device__ __forceinline__ void pair_of(int p, int N, int& i, int& j) {
    i = 0;
    int rem = p;
    while (rem >= N - 1 - i) {
        rem -= N - 1 - i;
        ++i;
    }
    j = i + 1 + rem;
}

// ---------------------------------------------------------------------------
// Barrier rows of one tick (build_barrier_constraints + fold_rows), owned by
// lanes: pair p by lane p % L; the two wall rows and two box sides of
// variable v by lane v; obstacle rows of robot i at slot o by lane 2i+(o&1).
// Global row indices follow the reference order (pairs, walls robot-major
// [x-min, x-max, y-min, y-max], obstacles robot-major, box hi/lo per
// variable), which is also the tie-break order of the QP scans.
// ---------------------------------------------------------------------------
template <class Real, int L, int MAXPAIR, int MAXOBS>
struct BarrierRows {
    int N, n, P, off_obs, off_box;
    int pi[MAXPAIR], pj[MAXPAIR];
    Real pgx[MAXPAIR], pgy[MAXPAIR], ph[MAXPAIR];
    Real wlo, whi, cap;
    int nob;
    Real ogx[MAXOBS > 0 ? MAXOBS : 1], ogy[MAXOBS > 0 ? MAXOBS : 1], oh[MAXOBS > 0 ? MAXOBS : 1];
    int oslot[MAXOBS > 0 ? MAXOBS : 1];           // obstacle index o (row order robot-major, then o)
    Real ocx[MAXOBS > 0 ? MAXOBS : 1], ocy[MAXOBS > 0 ? MAXOBS : 1], or2[MAXOBS > 0 ? MAXOBS : 1];
    unsigned active;

    __device__ __forceinline__ void consider(Real val, int idx, Real& worst, int& p) const {
        if (val > worst || (val == worst && p >= 0 && idx < p)) {
            worst = val;
            p = idx;
        }
    }

    __device__ __forceinline__ void scan(const Group<L>& g, Real u, Real& worst, int& p) const {
        const int lane = g.lane;
#pragma unroll
        for (int s = 0; s < MAXPAIR; ++s) {
            const int pidx = lane + s * L;
            const bool has = pidx < P;
            const Real uxi = g.shfl(u, 2 * pi[s]);
            const Real uyi = g.shfl(u, 2 * pi[s] + 1);
            const Real uxj = g.shfl(u, 2 * pj[s]);
            const Real uyj = g.shfl(u, 2 * pj[s] + 1);
            if (has && !((active >> s) & 1u))
                consider(pgx[s] * (uxj - uxi) + pgy[s] * (uyj - uyi) - ph[s], pidx, worst, p);
        }
        if (lane < n) {
            const int lo_idx = P + 4 * (lane >> 1) + 2 * (lane & 1);
            if (!((active >> MAXPAIR) & 1u)) consider(-u - wlo, lo_idx, worst, p);
            if (!((active >> (MAXPAIR + 1)) & 1u)) consider(u - whi, lo_idx + 1, worst, p);
            if (!((active >> (MAXPAIR + 2)) & 1u)) consider(u - cap, off_box + 2 * lane, worst, p);
            if (!((active >> (MAXPAIR + 3)) & 1u)) consider(-u - cap, off_box + 2 * lane + 1, worst, p);
        }
        if (MAXOBS > 0) {
            const Real ux = g.shfl(u, lane & ~1);
            const Real uy = g.shfl(u, (lane | 1) < L ? (lane | 1) : lane);
#pragma unroll
            for (int t = 0; t < (MAXOBS > 0 ? MAXOBS : 1); ++t) {
                if (t < nob && !((active >> (MAXPAIR + 4 + t)) & 1u))
                    consider(ogx[t] * ux + ogy[t] * uy - oh[t],
                             off_obs + (lane >> 1) * MRSIM_MAX_SLOTS + oslot[t], worst, p);
            }
        }
    }

    __device__ __forceinline__ void fetch(const Group<L>& g, int p, Real& gv, Real& hp) const {
        const int lane = g.lane;
        const int rv = lane >> 1, ax = lane & 1;
        if (p < P) {
            const int owner = p & (L - 1), s = p / L;
            Real gx = 0, gy = 0, h = 0;
            int ij = 0;
#pragma unroll
            for (int t = 0; t < MAXPAIR; ++t)
                if (t == s) {
                    gx = pgx[t];
                    gy = pgy[t];
                    h = ph[t];
                    ij = pi[t] | (pj[t] << 8);
                }
            gx = g.shfl(gx, owner);
            gy = g.shfl(gy, owner);
            h = g.shfl(h, owner);
            ij = g.shfl(ij, owner);
            const int i = ij & 0xff, j = ij >> 8;
            const Real comp = ax ? gy : gx;
            gv = (rv == j) ? comp : ((rv == i) ? -comp : Real(0));
            hp = h;
        } else if (p < off_obs) {
            const int q = p - P;
            const int owner = 2 * (q >> 2) + ((q & 3) >> 1);
            const bool hi = q & 1;
            hp = g.shfl(hi ? whi : wlo, owner);
            gv = (lane == owner) ? (hi ? Real(1) : Real(-1)) : Real(0);
        } else if (p < off_box) {
            const int q = p - off_obs;
            const int i = q / MRSIM_MAX_SLOTS, o = q % MRSIM_MAX_SLOTS;
            const int owner = 2 * i + (o & 1);
            Real gx = 0, gy = 0, h = 0;
#pragma unroll
            for (int t = 0; t < (MAXOBS > 0 ? MAXOBS : 1); ++t)
                if (t < nob && oslot[t] == o) {
                    gx = ogx[t];
                    gy = ogy[t];
                    h = oh[t];
                }
            gx = g.shfl(gx, owner);
            gy = g.shfl(gy, owner);
            hp = g.shfl(h, owner);
            gv = (rv == i) ? (ax ? gy : gx) : Real(0);
        } else {
            const int q = p - off_box;
            const int v0 = q >> 1;
            const bool lo = q & 1;
            gv = (lane == v0) ? (lo ? Real(-1) : Real(1)) : Real(0);
            hp = cap;
        }
    }

    __device__ __forceinline__ void set_active(const Group<L>& g, int p, bool on) {
        const int lane = g.lane;
        int owner, bit;
        if (p < P) {
            owner = p & (L - 1);
            bit = p / L;
        } else if (p < off_obs) {
            const int q = p - P;
            owner = 2 * (q >> 2) + ((q & 3) >> 1);
            bit = MAXPAIR + (q & 1);
        } else if (p < off_box) {
            const int q = p - off_obs;
            const int o = q % MRSIM_MAX_SLOTS;
            owner = 2 * (q / MRSIM_MAX_SLOTS) + (o & 1);
            bit = MAXPAIR + 4;
#pragma unroll
            for (int t = 0; t < (MAXOBS > 0 ? MAXOBS : 1); ++t)
                if (t < nob && oslot[t] == o) bit = MAXPAIR + 4 + t;
        } else {
            const int q = p - off_box;
            owner = q >> 1;
            bit = MAXPAIR + 2 + (q & 1);
        }
        if (lane == owner) {
            if (on) active |= 1u << bit;
            else active &= ~(1u << bit);
        }
    }
};


// One safety-filter evaluation (apply_barrier, barrier.hpp:132-205) for the
// group's robots: u_nom = uni_to_si(nominal), rows at the projected points,
// QP, infeasible -> zero commands, else map back with a uniform scale.
// Returns kQpOptimal/kQpIterLimit (commands set), kQpInfeasible (zeroed), or
// -1 for coincident projected points (domain_error, barrier.hpp:73-74).
template <class Real, int L, int MAXPAIR, int MAXOBS>
__device__ int barrier_filter(const Group<L>& g, BarrierRows<Real, L, MAXPAIR, MAXOBS>& rows, const QpSmem<Real>& ws,
                              const PhysConsts<Real>& k, int n, int P, bool vlane, int ax, int ri, Real prx, Real pry,
                              Real cs, Real sn, Real nv, Real nw, int total_rows, Real& cv, Real& cw) {
    const int lane = g.lane;
    Real u = 0;  // u_nom = uni_to_si(clamped nominal) (controllers.hpp:59-65)
    if (vlane) u = ax ? (sn * nv + k.l * cs * nw) : (cs * nv - k.l * sn * nw);
    // rows at the projected points (barrier.hpp:57-121 + fold_rows qp.hpp:104-125)
    bool coincident = false;
#pragma unroll
    for (int s = 0; s < MAXPAIR; ++s) {
        const int pidx = lane + s * L;
        const Real xi = g.shfl(prx, 2 * rows.pi[s]), yi = g.shfl(pry, 2 * rows.pi[s]);
        const Real xj = g.shfl(prx, 2 * rows.pj[s]), yj = g.shfl(pry, 2 * rows.pj[s]);
        const Real dx = xi - xj, dy = yi - yj;
        const Real dist2 = dx * dx + dy * dy;
        if (pidx < P && dist2 < Real(1e-18)) coincident = true;
        const Real h = dist2 - k.r_eff2;
        const Real inv = Real(1) / dsqrt(Real(8) * dist2);
        rows.pgx[s] = Real(2) * dx * inv;
        rows.pgy[s] = Real(2) * dy * inv;
        rows.ph[s] = k.gamma * h * h * h * inv;
    }
    if (g.any(coincident)) return -1;
    {
        const Real coord = ax ? pry : prx;
        const Real lo_h = coord - (ax ? k.wall_ymin : k.wall_xmin);
        const Real hi_h = (ax ? k.wall_ymax : k.wall_xmax) - coord;
        rows.wlo = k.gamma * lo_h * lo_h * lo_h;
        rows.whi = k.gamma * hi_h * hi_h * hi_h;
    }
    if (MAXOBS > 0) {
#pragma unroll
        for (int t = 0; t < (MAXOBS > 0 ? MAXOBS : 1); ++t) {
            if (t < rows.nob) {
                const Real dx = prx - rows.ocx[t];
                const Real dy = pry - rows.ocy[t];
                const Real h = dx * dx + dy * dy - rows.or2[t];
                const Real nrm = dsqrt(Real(4) * dx * dx + Real(4) * dy * dy);
                const Real gh = k.gamma * h * h * h;
                if (nrm < Real(1e-14)) {
                    rows.ogx[t] = 0;
                    rows.ogy[t] = 0;
                    rows.oh[t] = gh;
                } else {
                    rows.ogx[t] = Real(-2) * dx / nrm;
                    rows.ogy[t] = Real(-2) * dy / nrm;
                    rows.oh[t] = gh / nrm;
                }
            }
        }
    }
    rows.active = 0;
    const int status = qp_solve_group<Real, L>(g, rows, ws, n, u, total_rows, 0, k.tol, nullptr);
    if (status == kQpInfeasible) {  // barrier.hpp:178-182
        cv = 0;
        cw = 0;
        return status;
    }
    // map back + uniform scale (barrier.hpp:189-204)
    const Real ux = g.shfl(u, 2 * ri), uy = g.shfl(u, 2 * ri + 1);
    const Real mv = cs * ux + sn * uy;
    const Real mw = (-sn * ux + cs * uy) / k.l;
    Real scale = 1;
    if (vlane) {
        if (dabs(mv) > k.v_max) scale = dmin(scale, k.v_max / dabs(mv));
        if (dabs(mw) > k.w_max) scale = dmin(scale, k.w_max / dabs(mw));
    }
    scale = g.min(scale);
    cv = mv * scale;
    cw = mw * scale;
    return status;
}

template <int L>
struct LaneCfg;
template <>
struct LaneCfg<8> { static constexpr int kMaxN = 4, kMaxPair = 1; };
template <>
struct LaneCfg<16> { static constexpr int kMaxN = 8, kMaxPair = 2; };
template <>
struct LaneCfg<32> { static constexpr int kMaxN = 16, kMaxPair = 4; };

template <int TASK>
struct TaskCfg { static constexpr int kMaxObs = (TASK == MRSIM_TASK_RWARE) ? MRSIM_MAX_SLOTS / 2 : 0; };

// Shared-memory layout of one group.
template <class Real>
struct GroupSmem {
    QpSmem<Real> qp;
    Real *xs, *ys, *ts, *tf;
    int* ti;
    int* misc;
    static __host__ __device__ int bytes(int n, int N) {
        const int reals = QpSmem<Real>::reals(n) + 3 * N + kTfMax;
        const int ints = QpSmem<Real>::ints(n) + kTiMax + 4;
        int b = reals * static_cast<int>(sizeof(Real)) + ints * 4;
        return (b + 15) & ~15;
    }
    __device__ void carve(unsigned char* base, int n, int N) {
        Real* r = reinterpret_cast<Real*>(base);
        int* ib = reinterpret_cast<int*>(r + QpSmem<Real>::reals(n) + 3 * N + kTfMax);
        qp.carve(r, ib, n);
        xs = r + QpSmem<Real>::reals(n);
        ys = xs + N;
        ts = ys + N;
        tf = ts + N;
        ti = ib + QpSmem<Real>::ints(n);
        misc = ti + kTiMax;
    }
};

template <class Real>
__device__ __forceinline__ Real wrap_angle_dev(Real t) {  // core.hpp:102-108
    Real r = remainder(t, Consts<Real>::two_pi);
    if (r <= -Consts<Real>::pi) r += Consts<Real>::two_pi;
    return r;
}

// ---------------------------------------------------------------------------
// The fused step kernel. Persistent grid-stride loop over environments.
// ---------------------------------------------------------------------------
template <class Real, int L, int TASK>
__global__ void __launch_bounds__(256) step_kernel(const __grid_constant__ StepParams<Real> p) {
    constexpr int MAXPAIR = LaneCfg<L>::kMaxPair;
    constexpr int MAXOBS = TaskCfg<TASK>::kMaxObs;
    if (*p.err != ~0ull) return;  // sticky device error: later steps are no-ops

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Group<L> g;
    const int lane = g.lane;
    const int gpb = blockDim.x / L;
    const int gib = threadIdx.x / L;
    const mrsim_cfg& c = p.c;
    const int N = p.N, n = p.n, P = p.P;
    GroupSmem<Real> sm;
    sm.carve(smem_raw + gib * p.smem_bytes_per_group, n, N);

    // lane -> robot / axis
    const bool vlane = lane < n;
    const int ri = vlane ? (lane >> 1) : 0;
    const int ax = lane & 1;

    BarrierRows<Real, L, MAXPAIR, MAXOBS> rows;
    rows.N = N;
    rows.n = n;
    rows.P = P;
    rows.off_obs = P + 4 * N;
    rows.off_box = rows.off_obs + N * MRSIM_MAX_SLOTS;
    rows.cap = p.k.cap;
#pragma unroll
    for (int s = 0; s < MAXPAIR; ++s) {
        const int pidx = lane + s * L;
        int i = 0, j = 0;
        if (pidx < P) pair_of(pidx, N, i, j);
        rows.pi[s] = i;
        rows.pj[s] = j;
    }
    const int total_rows_base = P + 4 * N + 2 * n;
    const EnvView<Real> view{sm.xs, sm.ys, sm.ts, sm.tf, sm.ti, N};

    for (long long e = static_cast<long long>(blockIdx.x) * gpb + gib; e < p.B;
         e += static_cast<long long>(gridDim.x) * gpb) {
        // ---- load ----
        const int step_index = p.in.step_index[e];
        const uint64_t key = p.in.key[e];
        Real x = 0, y = 0, th = 0;
        if (vlane) {
            x = p.in.px[e * N + ri];
            y = p.in.py[e * N + ri];
            th = p.in.pt[e * N + ri];
        }
        for (int f = lane; f < p.nf; f += L) sm.tf[f] = p.in.tf[static_cast<long long>(f) * p.B + e];
        for (int w = lane; w < p.ni; w += L) sm.ti[w] = p.in.ti[static_cast<long long>(w) * p.B + e];
        g.sync();

        // ---- actions (validate_actions, batch.hpp:226-237) ----
        int act = 0;
        if (vlane) {
            act = p.actions ? static_cast<int>(p.actions[e * N + ri])
                            : policy_action(p.in.pkey[e], step_index, ri);
        }
        const unsigned badm = g.ballot(vlane && (act < 0 || act >= 5));
        if (badm) {
            const int bl = __ffs(badm) - 1;
            const int bad_act = g.shfl(act, bl);
            if (lane == 0) {
                report_error(p.err, e, bl >> 1, kErrInvalidAction, bad_act);
                *p.err_serial = p.serial;
            }
            g.sync();
            continue;
        }

        // ---- waypoints (Scenario::waypoints + action_to_waypoint) ----
        const uint64_t skey = fork_key(key, 1ull + static_cast<uint64_t>(step_index));  // step_stream
        Real wpx = x, wpy = y;
        if (vlane) {
            const Real ss = step_size_of<TASK, Real>(c, sm.ti, ri, x, y);
            const Real dxa = (act == 3) ? Real(-1) : ((act == 4) ? Real(1) : Real(0));
            const Real dya = (act == 1) ? Real(1) : ((act == 2) ? Real(-1) : Real(0));
            wpx = x + dxa * ss;
            wpy = y + dya * ss;
            if (c.action_noise_scale > 0.0) {
                const double half = c.action_noise_scale * static_cast<double>(ss);
                Rng nr{skey, static_cast<uint64_t>(2 * ri)};
                wpx += static_cast<Real>(nr.uniform(-half, half));
                wpy += static_cast<Real>(nr.uniform(-half, half));
            }
            wpx = dclamp(wpx, -p.k.hw, p.k.hw);
            wpy = dclamp(wpy, -p.k.hh, p.k.hh);
        }

        // ---- static obstacles (Scenario::add_obstacles, rware.hpp:54-68) ----
        int n_obs_rows = 0;
        if (MAXOBS > 0) {
            const int S = c.layout.rware_num_slots;
            unsigned carriers = 0;
            for (int i = 0; i < N; ++i) carriers |= (ti_byte(sm.ti, S + i) != 0 ? 1u : 0u) << i;
            rows.nob = 0;
            if (carriers != 0u) {
                int staged = 0;
                for (int o = 0; o < S; ++o) staged += ti_byte(sm.ti, o) != 0 ? 1 : 0;
                n_obs_rows = staged * __popc(carriers);
                if (vlane && ((carriers >> ri) & 1u)) {
                    int cnt = 0;
                    for (int o = ax; o < S; o += 2) {
                        if (ti_byte(sm.ti, o) == 0) continue;
#pragma unroll
                        for (int t = 0; t < (MAXOBS > 0 ? MAXOBS : 1); ++t)
                            if (t == cnt) {
                                rows.oslot[t] = o;
                                rows.ocx[t] = Real(c.layout.rware_slots[2 * o]);
                                rows.ocy[t] = Real(c.layout.rware_slots[2 * o + 1]);
                                rows.or2[t] = p.k.obs_r_eff2;
                            }
                        ++cnt;
                    }
                    rows.nob = cnt < MAXOBS ? cnt : MAXOBS;
                }
            }
        }
        const int total_rows = total_rows_base + n_obs_rows;

        // ---- physics ticks ----
        Real min_dist = p.in.min_dist[e];
        int qp_inf = p.in.qp_inf[e];
        bool collision = false;
        for (int tick = 0; tick < p.c.sub_steps; ++tick) {
            Real sn, cs;
            dsincos(th, &sn, &cs);
            const Real prx = x + cs * p.k.l;  // projected_point (controllers.hpp:34-36)
            const Real pry = y + sn * p.k.l;
            // nominal command (batch.hpp:183-191, controllers.hpp:39-55, 86-92)
            Real nv = 0, nw = 0;
            if (!(wpx == x && wpy == y)) {
                Real ux = p.k.k_pos * (wpx - prx);
                Real uy = p.k.k_pos * (wpy - pry);
                const Real nrm = dhypot(ux, uy);
                if (!(nrm <= p.k.si_max || nrm == Real(0))) {
                    const Real sc = p.k.si_max / nrm;
                    ux *= sc;
                    uy *= sc;
                }
                nv = dclamp(cs * ux + sn * uy, -p.k.v_max, p.k.v_max);
                nw = dclamp((-sn * ux + cs * uy) / p.k.l, -p.k.w_max, p.k.w_max);
            }
            Real cv = nv, cw = nw;
            if (c.barrier_enabled) {
                const int bs = barrier_filter<Real, L>(g, rows, sm.qp, p.k, n, P, vlane, ax, ri, prx, pry, cs, sn,
                                                       nv, nw, total_rows, cv, cw);
                if (bs < 0) {
                    if (lane == 0) {
                        report_error(p.err, e, 0, kErrCoincident);
                        *p.err_serial = p.serial;
                    }
                    break;
                }
                if (bs == kQpInfeasible) ++qp_inf;
            }
            // unicycle Euler step + wrap + arena clamp (core.hpp:112-118, batch.hpp:199-203)
            x = x + cv * cs * p.k.dt;
            y = y + cv * sn * p.k.dt;
            const Real tn = th + cw * p.k.dt;
            if (vlane && !isfinite(tn)) {
                report_error(p.err, e, ri, kErrNonFinite);
                *p.err_serial = p.serial;
            }
            th = wrap_angle_dev(tn);
            x = dclamp(x, -p.k.hw, p.k.hw);
            y = dclamp(y, -p.k.hh, p.k.hh);
            // collision check (batch.hpp:204-209)
            if (N > 1) {
                Real md = Consts<Real>::inf;
#pragma unroll
                for (int s = 0; s < MAXPAIR; ++s) {
                    const int pidx = lane + s * L;
                    const Real xi = g.shfl(x, 2 * rows.pi[s]), yi = g.shfl(y, 2 * rows.pi[s]);
                    const Real xj = g.shfl(x, 2 * rows.pj[s]), yj = g.shfl(y, 2 * rows.pj[s]);
                    if (pidx < P) md = dmin(md, dhypot(xi - xj, yi - yj));
                }
                md = g.min(md);
                min_dist = dmin(min_dist, md);
                collision = collision || md < p.k.coll_r;
            }
        }

        // ---- stage final poses, transition, bookkeeping (lane 0) ----
        if (vlane && ax == 0) {
            sm.xs[ri] = x;
            sm.ys[ri] = y;
            sm.ts[ri] = th;
        }
        g.sync();
        int done = 0;
        if (lane == 0) {
            Real metric = p.in.metric[e];
            int success = p.in.success[e];
            int collisions = p.in.collisions[e];
            Real ep_return = p.in.ep_return[e];
            Rng trng{skey, c.action_noise_scale > 0.0 ? static_cast<uint64_t>(2 * N) : 0ull};
            EnvView<Real> v = view;
            Real reward = transition_task<TASK, Real>(c, v, trng, metric);
            if (collision) {
                collisions += 1;
                reward += Real(c.coef[MRSIM_COEF_VIOLATION]);
            }
            const int new_step = step_index + 1;
            done = new_step >= c.max_steps ? 1 : 0;
            if (done) finalize_task<TASK, Real>(c, v, metric, success);
            ep_return += reward;
            if (p.reward) p.reward[e] = static_cast<float>(reward);
            if (p.reward64) p.reward64[e] = static_cast<double>(reward);
            if (p.done) p.done[e] = static_cast<uint8_t>(done);
            if (done && new_step == c.max_steps) {  // EpisodeStats (harness.hpp:277-285)
                p.st.episodes[e] += 1;
                p.st.ret[e] += static_cast<double>(ep_return);
                p.st.ret_sq[e] += static_cast<double>(ep_return) * static_cast<double>(ep_return);
                p.st.metric[e] += static_cast<double>(metric);
                p.st.success[e] += success ? 1.0 : 0.0;
                p.st.collisions[e] += collisions;
                p.st.qp_inf[e] += qp_inf;
                p.st.min_dist[e] = fmin(p.st.min_dist[e], static_cast<double>(min_dist));
            }
            sm.misc[0] = done;
            // publish bookkeeping through smem-free registers of lane 0 (stored below)
            p.out.step_index[e] = new_step;
            p.out.collisions[e] = collisions;
            p.out.qp_inf[e] = qp_inf;
            p.out.success[e] = success;
            p.out.metric[e] = metric;
            p.out.min_dist[e] = min_dist;
            p.out.ep_return[e] = ep_return;
            p.out.key[e] = key;
            p.out.seed[e] = p.in.seed[e];
            p.out.pkey[e] = p.in.pkey[e];
            p.out.episode[e] = p.in.episode[e];
        }
        g.sync();
        done = sm.misc[0];

        // ---- observations (assemble_observations, batch.hpp:143-151) ----
        const int ND = N * p.D;
        if (p.obs) {
            float* o = p.obs + e * ND;
            for (int q = lane; q < ND; q += L) {
                const int r = q / p.D;
                o[q] = obs_feature<TASK, Real>(c, view, r, q - r * p.D, p.bdim);
            }
        }

        // ---- auto-reset (harness wave semantics, harness.hpp:227-232) ----
        if (p.auto_reset && done) {
            if (lane == 0) {
                const long long episode = p.in.episode[e] + p.episode_stride;
                const uint64_t seed = derive_episode_seed(p.root_seed, episode);
                const uint64_t nkey = key_from_seed(seed);
                ResetOut ro;
                int bad = 0;
                const int rerr = reset_task<TASK>(c, nkey, ro, &bad);
                if (rerr) {
                    report_error(p.err, e, bad, static_cast<unsigned>(rerr));
                    *p.err_serial = p.serial;
                }
                for (int i = 0; i < N; ++i) {
                    sm.xs[i] = static_cast<Real>(ro.x[i]);
                    sm.ys[i] = static_cast<Real>(ro.y[i]);
                    sm.ts[i] = static_cast<Real>(ro.th[i]);
                }
                for (int f = 0; f < p.nf; ++f) sm.tf[f] = static_cast<Real>(ro.tf[f]);
                for (int w = 0; w < p.ni; ++w) sm.ti[w] = ro.ti[w];
                p.out.step_index[e] = 0;
                p.out.collisions[e] = 0;
                p.out.qp_inf[e] = 0;
                p.out.success[e] = 0;
                p.out.metric[e] = 0;
                p.out.min_dist[e] = Consts<Real>::inf;
                p.out.ep_return[e] = 0;
                p.out.key[e] = nkey;
                p.out.seed[e] = seed;
                p.out.pkey[e] = policy_key_of(seed);
                p.out.episode[e] = episode;
            }
            g.sync();
            if (p.next_obs) {
                float* o = p.next_obs + e * ND;
                for (int q = lane; q < ND; q += L) {
                    const int r = q / p.D;
                    o[q] = obs_feature<TASK, Real>(c, view, r, q - r * p.D, p.bdim);
                }
            }
        }

        // ---- store ----
        for (int i = lane; i < N; i += L) {
            p.out.px[e * N + i] = sm.xs[i];
            p.out.py[e * N + i] = sm.ys[i];
            p.out.pt[e * N + i] = sm.ts[i];
        }
        for (int f = lane; f < p.nf; f += L) p.out.tf[static_cast<long long>(f) * p.B + e] = sm.tf[f];
        for (int w = lane; w < p.ni; w += L) p.out.ti[static_cast<long long>(w) * p.B + e] = sm.ti[w];
        g.sync();
    }
}

// ---------------------------------------------------------------------------
// Reset kernel: one thread per env (reset_env, batch.hpp:153-160), then
// the reset observations. Seeds either explicit or derived from episodes.
// ---------------------------------------------------------------------------
template <class Real>
struct ResetParams {
    mrsim_cfg c;
    DevState<Real> out;
    const uint64_t* seeds;  // [B] or nullptr -> derive_episode_seed(root, first_episode + e)
    uint64_t root_seed;
    long long first_episode;
    float* obs;
    unsigned long long* err;
    long long B;
    int N, D, bdim, nf, ni;
};

template <class Real, int TASK>
__global__ void __launch_bounds__(128) reset_kernel(const __grid_constant__ ResetParams<Real> p) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= p.B) return;
    const mrsim_cfg& c = p.c;
    const int N = p.N;
    long long episode = -1;
    uint64_t seed;
    if (p.seeds) {
        seed = p.seeds[e];
    } else {
        episode = p.first_episode + e;
        seed = derive_episode_seed(p.root_seed, episode);
    }
    const uint64_t key = key_from_seed(seed);
    ResetOut ro;
    int bad = 0;
    const int err = reset_task<TASK>(c, key, ro, &bad);
    if (err) report_error(p.err, e, bad, static_cast<unsigned>(err));
    Real xs[MRSIM_MAX_ROBOTS], ys[MRSIM_MAX_ROBOTS], ts[MRSIM_MAX_ROBOTS], tf[kTfMax];
    for (int i = 0; i < N; ++i) {
        xs[i] = static_cast<Real>(ro.x[i]);
        ys[i] = static_cast<Real>(ro.y[i]);
        ts[i] = static_cast<Real>(ro.th[i]);
        p.out.px[e * N + i] = xs[i];
        p.out.py[e * N + i] = ys[i];
        p.out.pt[e * N + i] = ts[i];
    }
    for (int f = 0; f < p.nf; ++f) {
        tf[f] = static_cast<Real>(ro.tf[f]);
        p.out.tf[static_cast<long long>(f) * p.B + e] = tf[f];
    }
    for (int w = 0; w < p.ni; ++w) p.out.ti[static_cast<long long>(w) * p.B + e] = ro.ti[w];
    p.out.step_index[e] = 0;
    p.out.key[e] = key;
    p.out.seed[e] = seed;
    p.out.pkey[e] = policy_key_of(seed);
    p.out.episode[e] = episode;
    p.out.collisions[e] = 0;
    p.out.qp_inf[e] = 0;
    p.out.success[e] = 0;
    p.out.metric[e] = 0;
    p.out.min_dist[e] = Consts<Real>::inf;
    p.out.ep_return[e] = 0;
    if (p.obs) {
        const EnvView<Real> v{xs, ys, ts, tf, ro.ti, N};
        float* o = p.obs + e * N * p.D;
        for (int r = 0; r < N; ++r)
            for (int q = 0; q < p.D; ++q) o[r * p.D + q] = obs_feature<TASK, Real>(c, v, r, q, p.bdim);
    }
}

// assemble_observations of the current state (batch.hpp:143-151), one group per env.
template <class Real, int L, int TASK>
__global__ void __launch_bounds__(256) observe_kernel(const __grid_constant__ mrsim_cfg c, DevState<Real> s, float* obs,
                                                      long long B, int N, int D, int bdim, int nf, int ni,
                                                      int smem_bytes_per_group) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Group<L> g;
    const int gib = threadIdx.x / L;
    const long long e = static_cast<long long>(blockIdx.x) * (blockDim.x / L) + gib;
    if (e >= B) return;
    GroupSmem<Real> sm;
    sm.carve(smem_raw + gib * smem_bytes_per_group, 2 * N, N);
    for (int i = g.lane; i < N; i += L) {
        sm.xs[i] = s.px[e * N + i];
        sm.ys[i] = s.py[e * N + i];
        sm.ts[i] = s.pt[e * N + i];
    }
    for (int f = g.lane; f < nf; f += L) sm.tf[f] = s.tf[static_cast<long long>(f) * B + e];
    for (int w = g.lane; w < ni; w += L) sm.ti[w] = s.ti[static_cast<long long>(w) * B + e];
    g.sync();
    const EnvView<Real> view{sm.xs, sm.ys, sm.ts, sm.tf, sm.ti, N};
    float* o = obs + e * N * D;
    for (int q = g.lane; q < N * D; q += L) {
        const int r = q / D;
        o[q] = obs_feature<TASK, Real>(c, view, r, q - r * D, bdim);
    }
}

// Harness random-policy actions for the current step of every env.
template <class Real>
__global__ void random_actions_kernel(const int32_t* step_index, const uint64_t* pkey, int N, long long B,
                                      int8_t* out) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= B * N) return;
    const long long e = t / N;
    const int r = static_cast<int>(t - e * N);
    out[t] = static_cast<int8_t>(policy_action(pkey[e], step_index[e], r));
}

}  // namespace mrsim_dev
