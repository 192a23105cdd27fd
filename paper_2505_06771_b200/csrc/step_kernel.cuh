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
// Lane r of a group of L = next_pow2(N) lanes carries robot r (its pose and
// its two QP variables); pair rows are spread over all lanes; reductions are
// shuffles. A warp steps 32/L environments in lockstep (group.cuh).
#pragma once

#include "group.cuh"
#include "mrsim_device.cuh"
#include "qp_group.cuh"
#include "tasks.cuh"

// 128-thread blocks per SM the register budget is sized for (measured on B200): 4 -> <= 128 regs
// for L <= 8 and for L = 16 with up to 3 pair slots (N <= 10: arctic +8 %, MT +13 % over 3 since
// the counted warm-start loops, profiles/r02/ab_l16_minblocks.log); 3 -> <= 168 regs for wider
// L = 16 teams (N > 10, which spill at 128) and for rware, whose obstacle rows spill at 128 regs
// (+21% / +18% at N = 4 / 6). Shared memory caps the bench configurations at 4 blocks anyway.
#ifndef MRSIM_RW_MINB
#define MRSIM_RW_MINB 3
#endif
#ifndef MRSIM_SMALL_MINB
#define MRSIM_SMALL_MINB 4
#endif
#ifndef MRSIM_MIN_BLOCKS
#define MRSIM_MIN_BLOCKS(L, MP, TASK) \
    ((L) >= 16 ? ((MP) <= 3 ? 4 : 3) : (TASK) == MRSIM_TASK_RWARE ? MRSIM_RW_MINB : MRSIM_SMALL_MINB)
#endif

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

// Per-env accumulators over completed episodes (single buffer, touched only on
// done steps), with a one-level undo log: a step that fails is rolled back by
// the host (step_batch is pure, batch.hpp:267), and so are the stats it had
// already accumulated for other envs (stats_rollback_kernel).
struct EnvStats {
    int32_t* episodes;
    double *ret, *ret_sq, *metric, *success, *min_dist;
    int64_t *collisions, *qp_inf;
    int32_t* u_episodes;  // undo log: the values before the last update, and its step serial
    double *u_ret, *u_ret_sq, *u_metric, *u_success, *u_min_dist;
    int64_t *u_collisions, *u_qp_inf;
    long long* upd_serial;
};

// EpisodeStats update of a finished episode (harness.hpp:277-285).
__device__ __forceinline__ void stats_commit(const EnvStats& st, long long e, long long serial, double ret,
                                             double metric, int success, int collisions, int qp_inf,
                                             double min_dist) {
    if (st.upd_serial[e] != serial) {  // first update of this launch (a rollout may finish several episodes)
        st.u_episodes[e] = st.episodes[e];
        st.u_ret[e] = st.ret[e];
        st.u_ret_sq[e] = st.ret_sq[e];
        st.u_metric[e] = st.metric[e];
        st.u_success[e] = st.success[e];
        st.u_min_dist[e] = st.min_dist[e];
        st.u_collisions[e] = st.collisions[e];
        st.u_qp_inf[e] = st.qp_inf[e];
        st.upd_serial[e] = serial;
    }
    st.episodes[e] += 1;
    st.ret[e] += ret;
    st.ret_sq[e] += ret * ret;
    st.metric[e] += metric;
    st.success[e] += success ? 1.0 : 0.0;
    st.collisions[e] += collisions;
    st.qp_inf[e] += qp_inf;
    st.min_dist[e] = fmin(st.min_dist[e], min_dist);
}

// Undo the stats updates of the failed step `serial`.
__global__ void stats_rollback_kernel(EnvStats st, long long serial, long long B);

// Derived constants: SimParams, gains, BarrierConfig with the projection
// inflation of apply_barrier (barrier.hpp:151-157, 173).
template <class Real>
struct PhysConsts {
    Real dt, v_max, w_max, si_max, hw, hh, coll_r, coll_r2, k_pos, l, inv_l, gamma, r_eff2, cap, obs_r_eff2, tol;
    Real wall_xmin, wall_xmax, wall_ymin, wall_ymax;
    Real k_rho, k_alpha, k_beta, pose_ptol, pose_htol;  // pose controller (controllers.hpp:18-23)
};

template <class Real>
struct StepParams {
    mrsim_cfg c;
    DevState<Real> in, out;
    EnvStats st;
    const int8_t* actions;     // [B][N] or nullptr (on-device random policy)
    const int32_t* actions32;  // [B][N] the host API's std::vector<int> actions, used when actions is null
    float* obs;             // [B][N][D] or nullptr
    float* reward;          // [B] or nullptr
    double* reward64;       // [B] or nullptr (host-API path: the reference's double team reward)
    uint8_t* done;          // [B] or nullptr
    float* next_obs;        // [B][N][D] or nullptr
    unsigned long long* err;
    long long* err_serial;
    unsigned* ticket;       // [2] warp-task counters, used by alternate steps (serial & 1)
    long long serial;
    unsigned* exit_count;              // warps of this launch finished (err_epilogue; self-resetting)
    unsigned long long* err_host;      // pinned [error word, serial] written by the last warp, or nullptr
    long long B;
    long long e_begin, e_end;  // env range of this launch (the host API pipelines chunks of a step)
    int N, n, P, D, bdim, nf, ni;
    int auto_reset;
    int n_steps;               // consecutive steps per launch (1: mrsim_step; > 1: mrsim_rollout)
    long long obs_step_stride;  // floats between consecutive steps' obs blocks (rollout outputs)
    uint64_t root_seed;
    long long episode_stride;
    int smem_bytes_per_group;
    int obs_stage;  // floats per warp of the obs staging buffer after the group regions (0: direct stores)
    int obs_ws_stage;  // 1: stage each env's obs in its group's QP workspace instead (host-buffer steps)
    PhysConsts<Real> k;
    double prey_off[16];  // predator_prey candidate offsets (host-computed with the reference's libm)
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

template <int L>
struct LaneCfg {  // pair slots per lane for N <= L robots: ceil(L(L-1)/2 / L)
    static constexpr int kMaxPair = (L * (L - 1) / 2 + L - 1) / L;
};


// ---------------------------------------------------------------------------
// Barrier rows of one tick (build_barrier_constraints + fold_rows), owned by
// lanes: pair p by lane p % L; the four wall rows, the four box sides and
// the obstacle rows of robot r by lane r. Global row indices follow the
// reference order (pairs; walls robot-major [x-min, x-max, y-min, y-max];
// obstacles robot-major; box hi/lo per variable), which is also the
// tie-break order of the QP scans.
// active bits: [0,MP) pairs, MP+w walls, MP+4+b box (x-hi, x-lo, y-hi, y-lo), MP+8+t obstacles
// ---------------------------------------------------------------------------
// Row descriptor: components +(cx, cy) on robot r1 and -(cx, cy) on r0 for a
// pair row (r1 >= 0), or (cx, cy) on robot r0 (walls, box sides, obstacles); rhs h.
template <class Real>
struct BarrierDesc {
    int r0, r1;
    Real cx, cy, h;
};

template <class Real, int L, int MP, int MO>
struct BarrierRows {
    static constexpr int MO1 = MO > 0 ? MO : 1;
    // Row cache in shared memory, field-major [F][L] so lane-owned rows are
    // conflict-free and any lane can read the owner's row directly:
    //   pair slot s: fields 3s (gx), 3s+1 (gy), 3s+2 (rhs); walls: 3MP+w;
    //   obstacle slot t: 3MP+4+3t (gx), +1 (gy), +2 (rhs); then the lanes' current
    //   (ux, uy), published once per scan for the pair rows (cheaper than shuffles)
    static constexpr int kU = 3 * MP + 4 + 3 * MO;
    static constexpr int kFields = kU + 2;
    Real* rc;
    unsigned char* ptab;  // pair p -> robots (ptab[2p], ptab[2p+1]), shared by the block
    int N, P, off_obs, off_box;
    int npair;
    int pi[MP], pj[MP];
    Real cap;
    int nob;
    int oslot[MO1];
    // obstacle centres (x, y) by slot (stride ostride), radii by slot (+ oinfl) or one radius^2 for all
    const double* oxy;
    const double* orad;
    int ostride;
    double oinfl;
    Real or2u;
    unsigned active;
    bool valid;  // this lane carries a robot

    __device__ __forceinline__ Real& F(int f, int lane) const {
        MRSIM_DCHECK(f >= 0 && f < kFields && lane >= 0 && lane < L);
        return rc[f * L + lane];
    }
    __device__ __forceinline__ int dummy_row() const { return off_box; }

    // A lane scans its rows in increasing global index, so the reference's
    // strict `v > worst` (first maximal row wins) is exact within the lane;
    // the group argmax breaks cross-lane ties toward the lowest index.
    __device__ __forceinline__ static void consider(Real val, int idx, Real& worst, int& p) {
        if (val > worst) {
            worst = val;
            p = idx;
        }
    }
    __device__ __forceinline__ bool off(int bit) const { return !((active >> bit) & 1u); }

    __device__ __forceinline__ void scan(const Grp<L>& g, Real ux, Real uy, Real& worst, int& p) const {
        const int lane = g.lane;
        F(kU, lane) = ux;
        F(kU + 1, lane) = uy;
        Grp<L>::sync();
#pragma unroll
        for (int s = 0; s < MP; ++s) {  // branch-free: empty / active slots get -inf (their rows are finite)
            const Real uxi = F(kU, pi[s]), uyi = F(kU + 1, pi[s]);
            const Real uxj = F(kU, pj[s]), uyj = F(kU + 1, pj[s]);
            const Real v = F(3 * s, lane) * (uxj - uxi) + F(3 * s + 1, lane) * (uyj - uyi) - F(3 * s + 2, lane);
            consider((s < npair && off(s)) ? v : -Consts<Real>::inf, lane + s * L, worst, p);
        }
        if (valid) {
            const int w0 = P + 4 * lane;
            if (off(MP + 0)) consider(-ux - F(3 * MP + 0, lane), w0, worst, p);
            if (off(MP + 1)) consider(ux - F(3 * MP + 1, lane), w0 + 1, worst, p);
            if (off(MP + 2)) consider(-uy - F(3 * MP + 2, lane), w0 + 2, worst, p);
            if (off(MP + 3)) consider(uy - F(3 * MP + 3, lane), w0 + 3, worst, p);
            if (MO > 0) {
#pragma unroll
                for (int t = 0; t < MO1; ++t) {
                    const int f = 3 * MP + 4 + 3 * t;
                    if (t < nob && off(MP + 8 + t))
                        consider(F(f, lane) * ux + F(f + 1, lane) * uy - F(f + 2, lane),
                                 off_obs + lane * MRSIM_MAX_SLOTS + oslot[t], worst, p);
                }
            }
            // box sides (fold_rows qp.hpp:126-139): only reachable when |u| > cap
            if (dabs(ux) > cap || dabs(uy) > cap) {
                const int b0 = off_box + 4 * lane;
                if (off(MP + 4)) consider(ux - cap, b0, worst, p);
                if (off(MP + 5)) consider(-ux - cap, b0 + 1, worst, p);
                if (off(MP + 6)) consider(uy - cap, b0 + 2, worst, p);
                if (off(MP + 7)) consider(-uy - cap, b0 + 3, worst, p);
            }
        }
    }

    typedef BarrierDesc<Real> Desc;

    // Group-uniform descriptor of row p: pair rows read the owner lane's row
    // cache (shared memory broadcast); obstacle rows come from the owner's
    // registers through shuffles that run unconditionally (lockstep).
    __device__ __forceinline__ Desc describe(const Grp<L>& g, int p) const {
        Real ogx_b = 0, ogy_b = 0, oh_b = 0;
        if (MO > 0) {
            const int q = p - off_obs;
            const int o = q >= 0 ? q % MRSIM_MAX_SLOTS : 0;
            const int ow = q >= 0 ? (q / MRSIM_MAX_SLOTS) & (L - 1) : 0;
            int tt = 0;
#pragma unroll
            for (int u = 0; u < MO1; ++u)
                if (u < nob && oslot[u] == o) tt = u;
            const int t = g.shfl(tt, ow);
            const int f = 3 * MP + 4 + 3 * t;
            ogx_b = F(f, ow);
            ogy_b = F(f + 1, ow);
            oh_b = F(f + 2, ow);
        }
        MRSIM_DCHECK(p >= 0 && p <= off_box + 4 * N);
        Desc dsc;
        if (p < P) {  // pair (i, j): -(gx, gy) on i, +(gx, gy) on j
            const int owner = p & (L - 1), s = p / L;
            dsc.cx = F(3 * s, owner);
            dsc.cy = F(3 * s + 1, owner);
            dsc.h = F(3 * s + 2, owner);
            dsc.r0 = ptab[2 * p];
            dsc.r1 = ptab[2 * p + 1];
        } else if (p < off_obs) {  // wall w of robot r
            const int q = p - P, w = q & 3;
            dsc.r0 = q >> 2;
            dsc.r1 = -1;
            dsc.cx = (w == 0) ? Real(-1) : ((w == 1) ? Real(1) : Real(0));
            dsc.cy = (w == 2) ? Real(-1) : ((w == 3) ? Real(1) : Real(0));
            dsc.h = F(3 * MP + w, dsc.r0);
        } else if (p < off_box) {  // obstacle of robot r
            dsc.r0 = (p - off_obs) / MRSIM_MAX_SLOTS;
            dsc.r1 = -1;
            dsc.cx = ogx_b;
            dsc.cy = ogy_b;
            dsc.h = oh_b;
        } else {  // box side of variable v = 2r + axis
            const int q = p - off_box, b = q & 3;
            dsc.r0 = q >> 2;
            dsc.r1 = -1;
            dsc.cx = (b == 0) ? Real(1) : ((b == 1) ? Real(-1) : Real(0));
            dsc.cy = (b == 2) ? Real(1) : ((b == 3) ? Real(-1) : Real(0));
            dsc.h = cap;
        }
        return dsc;
    }
    __device__ __forceinline__ static void comp(const Desc& d, int lane, Real& cx, Real& cy) {
        const Real s = (d.r1 >= 0) ? ((lane == d.r1) ? Real(1) : ((lane == d.r0) ? Real(-1) : Real(0)))
                                   : ((lane == d.r0) ? Real(1) : Real(0));
        cx = s * d.cx;
        cy = s * d.cy;
    }
    __device__ __forceinline__ static bool touches(const Desc& d, int lane) { return lane == d.r0 || lane == d.r1; }
    __device__ __forceinline__ static Real rhs(const Desc& d) { return d.h; }
    // full dot product of two rows: sum over the robots they share
    __device__ __forceinline__ static Real dot(const Desc& a, const Desc& b) {
        const Real sa0 = (a.r1 >= 0) ? Real(-1) : Real(1), sb0 = (b.r1 >= 0) ? Real(-1) : Real(1);
        const Real cc = a.cx * b.cx + a.cy * b.cy;
        Real s = 0;
        if (a.r0 == b.r0) s += sa0 * sb0 * cc;
        if (a.r0 == b.r1) s += sa0 * cc;
        if (a.r1 >= 0 && a.r1 == b.r0) s += sb0 * cc;
        if (a.r1 >= 0 && a.r1 == b.r1) s += cc;
        return s;
    }

    // u of every robot of the group published in the row cache (the scan's slots), and a row's u
    __device__ __forceinline__ void publish_u(int lane, Real ux, Real uy) const {
        F(kU, lane) = ux;
        F(kU + 1, lane) = uy;
    }
    __device__ __forceinline__ Real dot_u(const Desc& d) const {
        const Real s0 = (d.r1 >= 0) ? Real(-1) : Real(1);
        Real v = s0 * (d.cx * F(kU, d.r0) + d.cy * F(kU + 1, d.r0));
        if (d.r1 >= 0) v += d.cx * F(kU, d.r1) + d.cy * F(kU + 1, d.r1);
        return v;
    }

    __device__ __forceinline__ void set_active(const Grp<L>& g, int p, bool on) {
        int owner, bit;
        if (p < P) {
            owner = p & (L - 1);
            bit = p / L;
        } else if (p < off_obs) {
            owner = (p - P) >> 2;
            bit = MP + ((p - P) & 3);
        } else if (p < off_box) {
            const int q = p - off_obs, o = q % MRSIM_MAX_SLOTS;
            owner = q / MRSIM_MAX_SLOTS;
            bit = MP + 8;
            if (MO > 0) {
#pragma unroll
                for (int t = 0; t < MO1; ++t)
                    if (t < nob && oslot[t] == o) bit = MP + 8 + t;
            }
        } else {
            owner = (p - off_box) >> 2;
            bit = MP + 4 + ((p - off_box) & 3);
        }
        if (g.lane == owner) active = on ? (active | (1u << bit)) : (active & ~(1u << bit));
    }
};

template <class Real, int L, int MP, int MO>
__device__ __forceinline__ void init_rows(BarrierRows<Real, L, MP, MO>& rows, Real* rc, unsigned char* ptab, int lane,
                                          int N, Real cap) {
    rows.rc = rc;
    rows.ptab = ptab;
    rows.N = N;
    rows.P = N * (N - 1) / 2;
    rows.off_obs = rows.P + 4 * N;
    rows.off_box = rows.off_obs + N * MRSIM_MAX_SLOTS;
    rows.cap = cap;
    rows.valid = lane < N;
    rows.nob = 0;
    rows.npair = 0;
    rows.oxy = nullptr;
    rows.orad = nullptr;
    rows.ostride = 2;
    rows.oinfl = 0.0;
    rows.or2u = Real(0);
#pragma unroll
    for (int s = 0; s < MP; ++s) {
        const int pidx = lane + s * L;
        int i = 0, j = 0;
        if (pidx < rows.P) {
            pair_of(pidx, N, i, j);
            rows.npair = s + 1;
            ptab[2 * pidx] = static_cast<unsigned char>(i);  // every group of the block writes the same table
            ptab[2 * pidx + 1] = static_cast<unsigned char>(j);
        }
        rows.pi[s] = i;
        rows.pj[s] = j;
    }
}

// One safety-filter evaluation (apply_barrier, barrier.hpp:132-205) for the
// group's robots: u_nom = uni_to_si(nominal), rows at the projected points,
// QP, infeasible -> zero commands, else map back with a uniform scale.
// Returns kQpOptimal/kQpIterLimit (commands set), kQpInfeasible (zeroed), or
// -1 for coincident projected points (domain_error, barrier.hpp:73-74).
template <class Real, int L, int MP, int MO, bool FAST, bool WARM = false>
__device__ __forceinline__ int barrier_filter(const Grp<L>& g, BarrierRows<Real, L, MP, MO>& rows,
                                              const QpWs<Real, BarrierDesc<Real>>& ws,
                              const PhysConsts<Real>& k, bool participate, Real prx, Real pry, Real cs, Real sn,
                              Real nv, Real nw, int total_rows, Real& cv, Real& cw, int* warm_k = nullptr) {
    const int lane = g.lane;
    const int n = 2 * rows.N;
    // u_nom = uni_to_si(clamped nominal) (controllers.hpp:59-65)
    Real ux = cs * nv - k.l * sn * nw;
    Real uy = sn * nv + k.l * cs * nw;
    if (!rows.valid) ux = uy = Real(0);
    // pair rows at the projected points (barrier.hpp:69-83 + fold_rows qp.hpp:104-125)
    bool coincident = false;
    constexpr int kU = BarrierRows<Real, L, MP, MO>::kU;  // publish the projected points (smem, not shuffles)
    rows.F(kU, lane) = prx;
    rows.F(kU + 1, lane) = pry;
    Grp<L>::sync();
#pragma unroll
    for (int s = 0; s < MP; ++s) {
        const Real xi = rows.F(kU, rows.pi[s]), yi = rows.F(kU + 1, rows.pi[s]);
        const Real xj = rows.F(kU, rows.pj[s]), yj = rows.F(kU + 1, rows.pj[s]);
        const Real dx = xi - xj, dy = yi - yj;
        const Real dist2 = dx * dx + dy * dy;
        if (s < rows.npair && dist2 < Real(1e-18)) coincident = true;
        const Real h = dist2 - k.r_eff2;
        // empty slots (s >= npair: i = j = 0, dist2 = 0) take 1 so rsqrt stays on its fast path
        // (rsqrt(0) calls the slow path: half a warp per tick at N = 4); their rows are never read
        const Real inv = rsqrt(Real(8) * (s < rows.npair ? dist2 : Real(1)));
        rows.F(3 * s, lane) = Real(2) * dx * inv;
        rows.F(3 * s + 1, lane) = Real(2) * dy * inv;
        rows.F(3 * s + 2, lane) = k.gamma * h * h * h * inv;
    }
    // walls (barrier.hpp:85-104)
    {
        const Real h0 = prx - k.wall_xmin, h1 = k.wall_xmax - prx;
        const Real h2 = pry - k.wall_ymin, h3 = k.wall_ymax - pry;
        rows.F(3 * MP + 0, lane) = k.gamma * h0 * h0 * h0;
        rows.F(3 * MP + 1, lane) = k.gamma * h1 * h1 * h1;
        rows.F(3 * MP + 2, lane) = k.gamma * h2 * h2 * h2;
        rows.F(3 * MP + 3, lane) = k.gamma * h3 * h3 * h3;
    }
    // static obstacles (barrier.hpp:106-119)
    if (MO > 0) {
#pragma unroll
        for (int t = 0; t < BarrierRows<Real, L, MP, MO>::MO1; ++t) {
            if (t < rows.nob) {
                const int o = rows.oslot[t] * rows.ostride;
                Real or2 = rows.or2u;
                if (rows.orad) {
                    const double r = rows.orad[o] + rows.oinfl;
                    or2 = Real(r * r);
                }
                const Real dx = prx - Real(rows.oxy[o]), dy = pry - Real(rows.oxy[o + 1]);
                const Real h = dx * dx + dy * dy - or2;
                const Real n2 = Real(4) * dx * dx + Real(4) * dy * dy;  // |row|^2 (fold_rows qp.hpp:104-125)
                const Real gh = k.gamma * h * h * h;
                const bool zero = n2 < Real(1e-28);                     // |row| < 1e-14
                const Real inv = zero ? Real(0) : rsqrt(n2);
                const int f = 3 * MP + 4 + 3 * t;
                rows.F(f, lane) = Real(-2) * dx * inv;
                rows.F(f + 1, lane) = Real(-2) * dy * inv;
                rows.F(f + 2, lane) = zero ? gh : gh * inv;
            }
        }
    }
    const bool bad = g.any(coincident);  // (the ballot also orders the row-cache writes before the QP reads)
    Grp<L>::sync();
    rows.active = 0;
    const int status = qp_solve<Real, L, FAST, WARM>(g, rows, ws, n, participate && !bad, ux, uy, total_rows, k.tol,
                                                     warm_k);
    // map back + uniform scale (barrier.hpp:186-204)
    const Real mv = cs * ux + sn * uy;
    const Real mw = (-sn * ux + cs * uy) * k.inv_l;
    Real scale = 1;
    if (rows.valid) {
        if (dabs(mv) > k.v_max) scale = dmin(scale, k.v_max / dabs(mv));
        if (dabs(mw) > k.w_max) scale = dmin(scale, k.w_max / dabs(mw));
    }
    scale = g.min(scale);
    const bool zero = status == kQpInfeasible;  // barrier.hpp:178-182
    cv = zero ? Real(0) : mv * scale;
    cw = zero ? Real(0) : mw * scale;
    (void)lane;
    return bad ? -1 : status;
}

// Shared-memory layout of one group: QP workspace, final-pose staging, task state.
template <class Real>
struct GroupSmem {
    QpWs<Real, BarrierDesc<Real>> qp;
    Real *xs, *ys, *ts, *tf, *rc;
    int *ti, *misc, *drones, *dcell;
    static constexpr int kG = 4 * MRSIM_GUARD_WORDS;  // checks builds: a guard behind each array
    static constexpr int kGuards = 9;
    static __host__ __device__ int rc_reals(int L, int MP, int MO) { return (3 * MP + 4 + 3 * MO + 2) * L; }
    static __host__ __device__ int bytes(int N, int nf, int ni, int L, int MP, int MO) {
        const int qb = (QpWs<Real, BarrierDesc<Real>>::bytes(2 * N) + 15) & ~15;
        const int reals = 3 * N + nf + rc_reals(L, MP, MO);
        const int ints = ni + 2 + N + 2 * N;  // task words, misc, drone list, drone cells
        const int b = qb + reals * static_cast<int>(sizeof(Real)) + ints * 4 + kGuards * kG;
        return (b + 15) & ~15;
    }
    __device__ void carve(unsigned char* base, int N, int nf, int ni, int rcr) {
        qp.carve(base, 2 * N);
#if MRSIM_GUARD_WORDS
        unsigned char* b = base + ((QpWs<Real, BarrierDesc<Real>>::bytes(2 * N) + 15) & ~15);
        auto take = [&](int bytes) {
            unsigned char* r = b;
            b += bytes + kG;
            return r;
        };
        xs = reinterpret_cast<Real*>(take(N * static_cast<int>(sizeof(Real))));
        ys = reinterpret_cast<Real*>(take(N * static_cast<int>(sizeof(Real))));
        ts = reinterpret_cast<Real*>(take(N * static_cast<int>(sizeof(Real))));
        tf = reinterpret_cast<Real*>(take(nf * static_cast<int>(sizeof(Real))));
        rc = reinterpret_cast<Real*>(take(rcr * static_cast<int>(sizeof(Real))));
        ti = reinterpret_cast<int*>(take(4 * ni));
        misc = reinterpret_cast<int*>(take(4 * 2));
        drones = reinterpret_cast<int*>(take(4 * N));
        dcell = reinterpret_cast<int*>(take(4 * 2 * N));
#else
        Real* r = reinterpret_cast<Real*>(base + ((QpWs<Real, BarrierDesc<Real>>::bytes(2 * N) + 15) & ~15));
        xs = r;
        ys = xs + N;
        ts = ys + N;
        tf = ts + N;
        rc = tf + nf;
        ti = reinterpret_cast<int*>(rc + rcr);
        misc = ti + ni;
        drones = misc + 2;
        dcell = drones + N;
#endif
    }
#if MRSIM_GUARD_WORDS
    // guard words behind each array (group lane 0 fills them per task and checks them at its end)
    __device__ unsigned* guard(int k, int N, int nf, int ni, int rcr) const {
        unsigned char* const ends[kGuards] = {
            reinterpret_cast<unsigned char*>(xs + N),  reinterpret_cast<unsigned char*>(ys + N),
            reinterpret_cast<unsigned char*>(ts + N),  reinterpret_cast<unsigned char*>(tf + nf),
            reinterpret_cast<unsigned char*>(rc + rcr), reinterpret_cast<unsigned char*>(ti + ni),
            reinterpret_cast<unsigned char*>(misc + 2), reinterpret_cast<unsigned char*>(drones + N),
            reinterpret_cast<unsigned char*>(dcell + 2 * N)};
        return reinterpret_cast<unsigned*>(ends[k / MRSIM_GUARD_WORDS]) + k % MRSIM_GUARD_WORDS;
    }
    __device__ void guards(bool fill, int N, int nf, int ni, int rcr) const {
        for (int k = 0; k < kGuards * MRSIM_GUARD_WORDS; ++k) {
            unsigned* w = guard(k, N, nf, ni, rcr);
            if (fill) *w = kGuardPattern;
            else MRSIM_DCHECK(*w == kGuardPattern);
        }
        for (int k = 0; k < 7 * MRSIM_GUARD_WORDS; ++k) {
            unsigned* w = qp.guard(2 * N, k);
            if (fill) *w = kGuardPattern;
            else MRSIM_DCHECK(*w == kGuardPattern);
        }
    }
#endif
};

// wrap_angle (core.hpp:102-108) for |t| < 3*pi: remainder(t, 2*pi) is t -/+ 2*pi,
// exact by Sterbenz, so this is bit-identical to the reference on the tick path.
// The far branch (|t| >= 3*pi: never reached from a tick, where |omega*dt| <= 0.12)
// is an out-of-line call so the inlined remainder() does not bloat the tick loops.
template <class Real>
__device__ __noinline__ Real wrap_angle_far(Real t) {
    return remainder(t, Consts<Real>::two_pi);
}
template <class Real>
__device__ __forceinline__ Real wrap_angle_dev(Real t) {
    Real r = t;
    if (dabs(r) >= Real(3) * Consts<Real>::pi) r = wrap_angle_far(t);
    else if (r > Consts<Real>::pi) r -= Consts<Real>::two_pi;
    else if (r < -Consts<Real>::pi) r += Consts<Real>::two_pi;
    if (r <= -Consts<Real>::pi) r += Consts<Real>::two_pi;
    return r;
}

#ifdef MRSIM_TASK_STATS
__device__ unsigned long long g_task_hist[64];
// per warp of the last launch: entry, first task start, last task end, busy time (globaltimer ns), tasks
constexpr int kWarpLogMax = 8192;
__device__ unsigned long long g_warp_log[kWarpLogMax * 5];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

template <class Real>
struct Real2 {
    Real a, b;
};

// unicycle_pose_controller (controllers.hpp:68-82): out of line, so the position
// controller's tick loop (the benchmark path) stays small in the instruction cache.
template <class Real>
__device__ __noinline__ Real2<Real> pose_nominal(const PhysConsts<Real>& K, Real x, Real y, Real th, Real wpx,
                                                 Real wpy, Real wh) {
    Real2<Real> out{Real(0), Real(0)};
    const Real dx = wpx - x, dy = wpy - y;
    const Real rho = dhypot(dx, dy);
    const Real herr = wrap_angle_dev(wh - th);
    if (!(rho < K.pose_ptol && dabs(herr) < K.pose_htol)) {
        const Real alpha = wrap_angle_dev(atan2(dy, dx) - th);
        const Real beta = wrap_angle_dev(wh - th - alpha);
        out.a = dclamp(K.k_rho * rho, -K.v_max, K.v_max);
        out.b = dclamp(K.k_alpha * alpha + K.k_beta * beta, -K.w_max, K.w_max);
    }
    return out;
}

// ---------------------------------------------------------------------------
// The fused step kernel. Persistent grid-stride loop; each warp steps 32/L
// environments in lockstep (ghost groups past the end compute but never store).
// ---------------------------------------------------------------------------
// Warm-start each tick's QP from the previous tick's active set (qp_solve WARM):
// a measured per-task choice (B200, fp64). MRSIM_QP_WARM = 0 off, 1 arctic only,
// 2 every task (A/B builds).
#ifndef MRSIM_QP_WARM
#define MRSIM_QP_WARM 1
#endif
__host__ __device__ constexpr bool qp_warm_order(int task) {
    return MRSIM_QP_WARM == 2 || (MRSIM_QP_WARM == 1 && task == MRSIM_TASK_ARCTIC_TRANSPORT);
}

// First-row QP fast path (qp_solve FAST): a measured choice (B200, fp64). It
// pays for groups of 4 (teams of up to 4 robots: navigation +6%, warehouse +7%,
// foraging +4%, rware neutral) and costs 2-4% for L = 8 (discovery / foraging
// N = 6); L = 16 is neutral.
__host__ __device__ constexpr bool qp_fast_first_row(int L) {
#ifdef MRSIM_QP_NO_FAST
    return false && L;
#endif
    return L == 4;
}

// Host-buffer obs staged in the group's QP workspace (StepParams::obs_ws_stage): compiled only into
// the tasks whose warp stage costs too much (capi.cu's rule picks it for arctic_transport and
// rware); in the others the extra branch alone cost 2-3 % (navigation, MT; profiles/r02/ab_ws_regress.log).
__host__ __device__ constexpr bool obs_ws_stage_task(int task) {
    return task == MRSIM_TASK_ARCTIC_TRANSPORT || task == MRSIM_TASK_RWARE;
}

// MULTI: the mrsim_rollout instantiation (p.n_steps steps per task); the single-step instantiation
// compiles the step loop away (the loop and the input-copy select cost 2-6 % when always present).
template <class Real, int L, int MP, int MO, int TASK, bool MULTI = false>
__device__ __forceinline__ void step_body(const StepParams<Real>& p) {
    constexpr int G = 32 / L;  // envs per warp
    // Dynamic warp tasks: a warp takes the next G consecutive envs from a counter. Step k
    // uses counter k & 1 and clears the other one for step k + 1 (stream order makes that
    // safe: step k - 1, its last user, has finished).
    if (MRSIM_DYN_SCHED && blockIdx.x == 0 && threadIdx.x == 0) p.ticket[(p.serial + 1) & 1] = 0u;
    if (*p.err != ~0ull) return;  // sticky device error: later steps are no-ops

    extern __shared__ __align__(16) unsigned char smem_raw[];
    const Grp<L> g;
    const int lane = g.lane;
    const int gpb = blockDim.x / L;
    const int gib = threadIdx.x / L;
    const mrsim_cfg& c = p.c;
    const int N = p.N;
    GroupSmem<Real> sm;
    sm.carve(smem_raw + gib * p.smem_bytes_per_group, N, p.nf, p.ni, GroupSmem<Real>::rc_reals(L, MP, MO));
    int* misc = sm.misc;
    MRSIM_DCHECK(reinterpret_cast<unsigned char*>(sm.dcell + 2 * N) + GroupSmem<Real>::kG <=
                 smem_raw + (gib + 1) * p.smem_bytes_per_group);
    int n_drones = 0;
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) n_drones = arctic_drones(c, sm.drones);

    const bool vl = lane < N;  // lane r carries robot r
    const int ri = vl ? lane : 0;

    BarrierRows<Real, L, MP, MO> rows;
    __shared__ unsigned char pair_tab[MRSIM_MAX_ROBOTS * (MRSIM_MAX_ROBOTS - 1)];
    init_rows(rows, sm.rc, pair_tab, lane, N, p.k.cap);
    rows.oxy = c.layout.rware_slots;  // rware shelves: one inflated radius (barrier.hpp:157)
    rows.or2u = p.k.obs_r_eff2;
    const int total_rows_base = rows.P + 4 * N + 4 * N;
    __shared__ double het_flat[MRSIM_MAX_ROBOTS * MRSIM_MAX_HET_COLS];  // het_augment, full team, feature order
    for (int k = threadIdx.x; k < c.het_rows * c.het_cols; k += blockDim.x) het_flat[k] = c.het[k / c.het_cols][k % c.het_cols];
    __syncthreads();
    const EnvView<Real> view{sm.xs, sm.ys, sm.ts, sm.tf, sm.ti, N, sm.drones, p.prey_off,
                             TASK == MRSIM_TASK_ARCTIC_TRANSPORT ? sm.dcell : nullptr, het_flat};
    const long long stride = static_cast<long long>(gridDim.x) * gpb;
#ifdef MRSIM_TASK_STATS
    const unsigned long long w_enter = gtimer();
    unsigned long long w_first = 0, w_last = 0, w_busy = 0, w_tasks = 0;
#endif

    auto next_task = [&](long long e_static) -> long long {
        if (!MRSIM_DYN_SCHED) return e_static;
        unsigned t = 0;
        if ((threadIdx.x & 31) == 0) t = atomicAdd(p.ticket + (p.serial & 1), 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        return p.e_begin + static_cast<long long>(t) * G;
    };
    for (long long e0 = next_task(p.e_begin + static_cast<long long>(blockIdx.x) * gpb + (gib & ~(G - 1)));
         e0 < p.e_end; e0 = next_task(e0 + stride)) {
        const long long e_real = e0 + (gib & (G - 1));
        const bool ghost = e_real >= p.e_end;
        const long long e = ghost ? p.e_end - 1 : e_real;
        MRSIM_DCHECK(e >= 0 && e < p.B);
#if MRSIM_GUARD_WORDS
        if (lane == 0) sm.guards(true, N, p.nf, p.ni, GroupSmem<Real>::rc_reals(L, MP, MO));
        Grp<L>::sync();
#endif
#ifdef MRSIM_TASK_STATS
        const long long t_task0 = clock64();
        const unsigned long long g_task0 = gtimer();
        if (w_first == 0) w_first = g_task0;
#endif
        // mrsim_rollout: n_steps consecutive steps of the task's envs in this launch. Step 0 reads
        // the input copy, later steps update the output copy in place (each env belongs to this
        // group alone), so the input copy stays untouched for the rollback of a failing launch.
        const int n_steps = MULTI ? p.n_steps : 1;
        for (int s = 0; s < n_steps; ++s) {
            const DevState<Real>& in = (MULTI && s > 0) ? p.out : p.in;
            float* const obs_s = p.obs ? p.obs + s * p.obs_step_stride : nullptr;
            float* const reward_s = p.reward ? p.reward + s * p.B : nullptr;
            uint8_t* const done_s = p.done ? p.done + s * p.B : nullptr;
            // ---- load ----
            const int step_index = in.step_index[e];
            const uint64_t key = in.key[e];
            Real x = in.px[e * N + ri], y = in.py[e * N + ri], th = in.pt[e * N + ri];
            for (int f = lane; f < p.nf; f += L) sm.tf[f] = in.tf[static_cast<long long>(f) * p.B + e];
            for (int w = lane; w < p.ni; w += L) sm.ti[w] = in.ti[static_cast<long long>(w) * p.B + e];
            Grp<L>::sync();

            // ---- actions (validate_actions, batch.hpp:226-237) ----
            int act = 0;
            if (vl)
                act = p.actions ? static_cast<int>(p.actions[e * N + ri])
                                : (p.actions32 ? p.actions32[e * N + ri] : policy_action(in.pkey[e], step_index, ri));
            const int bad_robot = g.first(vl && (act < 0 || act >= 5));
            const int bad_act = g.shfl(act, bad_robot < 0 ? 0 : bad_robot);
            if (bad_robot >= 0 && lane == 0 && !ghost) {
                report_error(p.err, e, bad_robot, kErrInvalidAction, bad_act);
                *p.err_serial = p.serial;
            }
            bool skip = ghost || bad_robot >= 0;  // compute in lockstep, never store

            // ---- waypoints (Scenario::waypoints + action_to_waypoint) ----
            const uint64_t skey = fork_key(key, 1ull + static_cast<uint64_t>(step_index));  // step_stream
            Real wpx = x, wpy = y;
            if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {  // actions ignored: the stored targets (random_waypoints.hpp:40-44)
                if (vl) {
                    wpx = sm.tf[2 * ri];
                    wpy = sm.tf[2 * ri + 1];
                }
            } else if (vl) {
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

            // goal headings for the pose controller (Scenario::waypoint_headings, batch.hpp:169-171)
            const bool pose_ctl = c.controller == MRSIM_CONTROLLER_UNICYCLE_POSE;
            Real wth = th;
            if (pose_ctl) {
                if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {
                    wth = sm.tf[2 * N + ri];  // random_waypoints.hpp:46-50
                } else {  // scenario.hpp:168-177
                    const Real ddx = wpx - x, ddy = wpy - y;
                    wth = dhypot(ddx, ddy) > Real(1e-12) ? atan2(ddy, ddx) : th;
                }
            }

            // ---- static obstacles (Scenario::add_obstacles, rware.hpp:54-68) ----
            int n_obs_rows = 0;
            if (MO > 0) {
                const int S = c.layout.rware_num_slots;
                unsigned carriers = 0;
                for (int i = 0; i < N; ++i) carriers |= (ti_byte(sm.ti, S + i) != 0 ? 1u : 0u) << i;
                rows.nob = 0;
                if (carriers != 0u) {
                    int staged = 0;
                    for (int o = 0; o < S; ++o) staged += ti_byte(sm.ti, o) != 0 ? 1 : 0;
                    n_obs_rows = staged * __popc(carriers);
                    if (vl && ((carriers >> ri) & 1u)) {
                        int cnt = 0;
                        for (int o = 0; o < S; ++o) {
                            if (ti_byte(sm.ti, o) == 0) continue;
#pragma unroll
                            for (int t = 0; t < BarrierRows<Real, L, MP, MO>::MO1; ++t)
                                if (t == cnt) {
                                    rows.oslot[t] = o;
                                }
                            ++cnt;
                        }
                        rows.nob = cnt;
                    }
                }
            }
            const int total_rows = total_rows_base + n_obs_rows;

            // ---- physics ticks ----
            Real min_dist = in.min_dist[e];
            Real min_d2 = Consts<Real>::inf;  // min squared pairwise distance over this step's ticks
            int qp_inf = in.qp_inf[e];
            bool collision = false;
            int warm_k = 0;  // QP warm entering order: the previous tick's active rows (none at a step's first tick)
            for (int tick = 0; tick < c.sub_steps; ++tick) {
                Real sn, cs;
                dsincos(th, &sn, &cs);
                const Real prx = x + cs * p.k.l;  // projected_point (controllers.hpp:34-36)
                const Real pry = y + sn * p.k.l;
                // nominal command (batch.hpp:183-191, controllers.hpp:39-55, 86-92)
                Real nv = 0, nw = 0;
                if (pose_ctl) {  // unicycle_pose_controller (controllers.hpp:68-82), out of line
                    const Real2<Real> c2 = pose_nominal<Real>(p.k, x, y, th, wpx, wpy, wth);
                    nv = c2.a;
                    nw = c2.b;
                } else if (!(wpx == x && wpy == y)) {
                    Real ux = p.k.k_pos * (wpx - prx);
                    Real uy = p.k.k_pos * (wpy - pry);
                    const Real nrm = dsqrt(ux * ux + uy * uy);
                    if (!(nrm <= p.k.si_max || nrm == Real(0))) {
                        const Real sc = p.k.si_max / nrm;
                        ux *= sc;
                        uy *= sc;
                    }
                    nv = dclamp(cs * ux + sn * uy, -p.k.v_max, p.k.v_max);
                    nw = dclamp((-sn * ux + cs * uy) * p.k.inv_l, -p.k.w_max, p.k.w_max);
                }
                Real cv = nv, cw = nw;
                if (c.barrier_enabled) {
                    const int bs = barrier_filter<Real, L, MP, MO, qp_fast_first_row(L), qp_warm_order(TASK)>(g, rows, sm.qp, p.k, !skip, prx, pry, cs, sn, nv, nw,
                                                           total_rows, cv, cw, qp_warm_order(TASK) ? &warm_k : nullptr);
                    if (bs < 0 && !skip) {
                        if (lane == 0) {
                            report_error(p.err, e, 0, kErrCoincident);
                            *p.err_serial = p.serial;
                        }
                        skip = true;
                    }
                    if (bs == kQpInfeasible) ++qp_inf;
                }
                // unicycle Euler step + wrap + arena clamp (core.hpp:112-118, batch.hpp:199-203)
                x = x + cv * cs * p.k.dt;
                y = y + cv * sn * p.k.dt;
                const Real tn = th + cw * p.k.dt;
                if (vl && !skip && !isfinite(tn)) {
                    report_error(p.err, e, ri, kErrNonFinite);
                    *p.err_serial = p.serial;
                }
                th = wrap_angle_dev(tn);
                x = dclamp(x, -p.k.hw, p.k.hw);
                y = dclamp(y, -p.k.hh, p.k.hh);
                // collision check (batch.hpp:204-209)
                if (N > 1) {  // squared distances; sqrt is monotone, so it is taken once per step
                    Real md2 = Consts<Real>::inf;
                    constexpr int kU = BarrierRows<Real, L, MP, MO>::kU;  // publish the poses (smem, not shuffles)
                    Grp<L>::sync();
                    rows.F(kU, lane) = x;
                    rows.F(kU + 1, lane) = y;
                    Grp<L>::sync();
#pragma unroll
                    for (int s = 0; s < MP; ++s) {
                        const Real xi = rows.F(kU, rows.pi[s]), yi = rows.F(kU + 1, rows.pi[s]);
                        const Real xj = rows.F(kU, rows.pj[s]), yj = rows.F(kU + 1, rows.pj[s]);
                        const Real dx = xi - xj, dy = yi - yj;
                        md2 = dmin(md2, s < rows.npair ? dx * dx + dy * dy : Consts<Real>::inf);
                    }
                    md2 = g.min(md2);
                    min_d2 = dmin(min_d2, md2);
                    collision = collision || md2 < p.k.coll_r2;
                }
            }

            min_dist = dmin(min_dist, dsqrt(min_d2));
            // ---- stage final poses, transition, bookkeeping (lane 0) ----
            if (vl) {
                sm.xs[ri] = x;
                sm.ys[ri] = y;
                sm.ts[ri] = th;
            }
            Grp<L>::sync();
            if (lane == 0) {
                Real metric = in.metric[e];
                int success = in.success[e];
                int collisions = in.collisions[e];
                Real ep_return = in.ep_return[e];
                // the transition continues the step stream after the waypoint noise draws
                Rng trng{skey, (c.action_noise_scale > 0.0 && TASK != MRSIM_TASK_RANDOM_WAYPOINTS)
                                   ? static_cast<uint64_t>(2 * N) : 0ull};
                EnvView<Real> v = view;
                Real reward = transition_task<TASK, Real>(c, v, trng, metric);
                if (collision) {
                    collisions += 1;
                    reward += Real(c.coef[MRSIM_COEF_VIOLATION]);
                }
                const int new_step = step_index + 1;
                const int done = new_step >= c.max_steps ? 1 : 0;
                if (done) finalize_task<TASK, Real>(c, v, metric, success);
                ep_return += reward;
                misc[0] = done;
                if (!skip) {
                    if (reward_s) reward_s[e] = static_cast<float>(reward);
                    if (p.reward64) p.reward64[e] = static_cast<double>(reward);
                    if (done_s) done_s[e] = static_cast<uint8_t>(done);
                    if (done && new_step == c.max_steps)  // EpisodeStats (harness.hpp:277-285)
                        stats_commit(p.st, e, p.serial, static_cast<double>(ep_return), static_cast<double>(metric),
                                     success, collisions, qp_inf, static_cast<double>(min_dist));
                    p.out.step_index[e] = new_step;
                    p.out.collisions[e] = collisions;
                    p.out.qp_inf[e] = qp_inf;
                    p.out.success[e] = success;
                    p.out.metric[e] = metric;
                    p.out.min_dist[e] = min_dist;
                    p.out.ep_return[e] = ep_return;
                    p.out.key[e] = key;
                    p.out.seed[e] = in.seed[e];
                    p.out.pkey[e] = in.pkey[e];
                    p.out.episode[e] = in.episode[e];
                }
            }
            Grp<L>::sync();
            const int done = misc[0];

            // ---- observations (assemble_observations, batch.hpp:143-151) ----
            if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) {  // each drone's cell once, not once per patch feature
                if (lane < n_drones) {
                    const int d = sm.drones[lane];
                    arctic_cell<Real>(c, sm.xs[d], sm.ys[d], sm.dcell[2 * lane], sm.dcell[2 * lane + 1]);
                }
                Grp<L>::sync();
            }
            const int ND = N * p.D;
            if (obs_s && p.obs_stage) {
                // the warp's G envs are consecutive: stage their obs, then store one contiguous block
                // (float4 stores when the block is 16-byte aligned: every store instruction writes
                // 512 contiguous bytes; else 128)
                float* wst = reinterpret_cast<float*>(smem_raw + gpb * p.smem_bytes_per_group) +
                             (threadIdx.x >> 5) * p.obs_stage;
                float* mine = wst + (gib & (G - 1)) * ND;
                MRSIM_DCHECK(((gib & (G - 1)) + 1) * ND <= p.obs_stage);
                for (int q = lane, r = lane / p.D, f = lane - (lane / p.D) * p.D; q < ND; q += L) {
                    mine[q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, f, p.bdim));
                    for (f += L; f >= p.D; f -= p.D) ++r;
                }
                __syncwarp();
                const long long left = p.e_end - e0;
                const int total = static_cast<int>(left < G ? left : G) * ND;
                float* dst = obs_s + e0 * ND;
                MRSIM_DCHECK(total <= p.obs_stage && e0 * ND + total <= p.B * ND);
                if (((e0 * ND) & 3) == 0 && (total & 3) == 0) {
                    const float4* src4 = reinterpret_cast<const float4*>(wst);
                    float4* dst4 = reinterpret_cast<float4*>(dst);
                    for (int k = threadIdx.x & 31; k < total / 4; k += 32) dst4[k] = src4[k];
                } else {
                    for (int k = threadIdx.x & 31; k < total; k += 32) dst[k] = wst[k];
                }
                __syncwarp();
            } else if (obs_ws_stage_task(TASK) && obs_s && p.obs_ws_stage) {
                // host-buffer steps whose warp stage would cost a resident block: each group stages
                // its env's obs in its own QP inverse-Gram matrix (dead after the ticks), and the warp
                // stores its consecutive envs' block as 8-byte pieces (256 contiguous bytes per store)
                float* mine = reinterpret_cast<float*>(sm.qp.S);
                MRSIM_DCHECK(ND * 4 <= 4 * N * N * static_cast<int>(sizeof(Real)) && (ND & 1) == 0);
                for (int q = lane, r = lane / p.D, f = lane - (lane / p.D) * p.D; q < ND; q += L) {
                    mine[q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, f, p.bdim));
                    for (f += L; f >= p.D; f -= p.D) ++r;
                }
                __syncwarp();
                const long long left = p.e_end - e0;
                const int half = ND / 2;  // float2 per env
                const int total2 = static_cast<int>(left < G ? left : G) * half;
                const unsigned char* wbase = smem_raw + (gib & ~(G - 1)) * p.smem_bytes_per_group;
                float2* dst2 = reinterpret_cast<float2*>(obs_s + e0 * ND);
                for (int k = threadIdx.x & 31; k < total2; k += 32) {
                    const int g2 = k / half;
                    dst2[k] = reinterpret_cast<const float2*>(wbase + g2 * p.smem_bytes_per_group)[k - g2 * half];
                }
                __syncwarp();
            } else if (obs_s && !skip) {
                float* o = obs_s + e * ND;
                for (int q = lane, r = lane / p.D, f = lane - (lane / p.D) * p.D; q < ND; q += L) {
                    o[q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, f, p.bdim));
                    for (f += L; f >= p.D; f -= p.D) ++r;
                }
            }

            // ---- auto-reset (harness wave semantics, harness.hpp:227-232) ----
            if (p.auto_reset && done && !skip) {
                if (lane == 0) {
                    const long long episode = in.episode[e] + p.episode_stride;
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
            }
            Grp<L>::sync();
            if (p.auto_reset && done && !skip && p.next_obs) {
                EnvView<Real> fresh = view;  // the drone-cell cache holds the terminal poses
                fresh.dcell = nullptr;
                float* o = p.next_obs + e * ND;
                for (int q = lane; q < ND; q += L) {
                    const int r = q / p.D;
                    o[q] = static_cast<float>(obs_feature<TASK, Real>(c, fresh, r, q - r * p.D, p.bdim));
                }
            }

            // ---- store ----
            if (!skip) {
                for (int i = lane; i < N; i += L) {
                    p.out.px[e * N + i] = sm.xs[i];
                    p.out.py[e * N + i] = sm.ys[i];
                    p.out.pt[e * N + i] = sm.ts[i];
                }
                for (int f = lane; f < p.nf; f += L) p.out.tf[static_cast<long long>(f) * p.B + e] = sm.tf[f];
                for (int w = lane; w < p.ni; w += L) p.out.ti[static_cast<long long>(w) * p.B + e] = sm.ti[w];
            }
            Grp<L>::sync();
        }  // rollout steps
#if MRSIM_GUARD_WORDS
        Grp<L>::sync();
        if (lane == 0) sm.guards(false, N, p.nf, p.ni, GroupSmem<Real>::rc_reals(L, MP, MO));
#endif
#ifdef MRSIM_TASK_STATS  // diagnostic builds: histogram of warp-task durations (log2 of SM cycles)
        if ((threadIdx.x & 31) == 0) {
            const long long dt = clock64() - t_task0;
            const int b = dt > 0 ? 63 - __clzll(dt) : 0;
            atomicAdd(&g_task_hist[b < 47 ? b : 47], 1ull);
            atomicAdd(&g_task_hist[48], static_cast<unsigned long long>(dt));
        }
        w_last = gtimer();
        w_busy += w_last - g_task0;
        ++w_tasks;
#endif
    }
#ifdef MRSIM_TASK_STATS
    {
        const unsigned wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
        if ((threadIdx.x & 31) == 0 && wid < kWarpLogMax) {
            unsigned long long* o = g_warp_log + 5 * wid;
            o[0] = w_enter;
            o[1] = w_first;
            o[2] = w_last;
            o[3] = w_busy;
            o[4] = w_tasks;
        }
    }
#endif
}

// Host-API steps: the last warp of the launch to finish copies the error word and its serial into
// the caller-visible pinned word (p.err_host), so the synchronous host step needs no separate
// device-to-host copy after the kernel (one stream operation, ~7 us, less per step).
template <class Real>
__device__ __forceinline__ void err_epilogue(const StepParams<Real>& p) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence();  // this warp's error reports are visible before it is counted
        const unsigned warps = gridDim.x * (blockDim.x >> 5);
        if (atomicAdd(p.exit_count, 1u) == warps - 1) {
            __threadfence();
            const unsigned long long w = *reinterpret_cast<volatile unsigned long long*>(p.err);
            p.err_host[1] = static_cast<unsigned long long>(*reinterpret_cast<volatile long long*>(p.err_serial));
            p.err_host[0] = w;
            __threadfence_system();
            *p.exit_count = 0u;  // ready for the next launch (stream order)
        }
    }
}

template <class Real, int L, int MP, int MO, int TASK, bool MULTI = false>
__global__ void __launch_bounds__(128, MRSIM_MIN_BLOCKS(L, MP, TASK)) step_kernel(const __grid_constant__ StepParams<Real> p) {
    step_body<Real, L, MP, MO, TASK, MULTI>(p);
    if (p.err_host) err_epilogue(p);
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
        int drones[MRSIM_MAX_ROBOTS];
        arctic_drones(c, drones);
        const EnvView<Real> v{xs, ys, ts, tf, ro.ti, N, drones, nullptr};
        float* o = p.obs + e * N * p.D;
        for (int r = 0; r < N; ++r)
            for (int q = 0; q < p.D; ++q) o[r * p.D + q] = static_cast<float>(obs_feature<TASK, Real>(c, v, r, q, p.bdim));
    }
}

// assemble_observations of the current state (batch.hpp:143-151), one thread per env.
template <class Real, int TASK>
__global__ void __launch_bounds__(128) observe_kernel(const __grid_constant__ mrsim_cfg c, DevState<Real> s, float* obs,
                                                      long long B, int N, int D, int bdim, int nf, int ni) {
    const long long e = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= B) return;
    Real xs[MRSIM_MAX_ROBOTS], ys[MRSIM_MAX_ROBOTS], ts[MRSIM_MAX_ROBOTS], tf[kTfMax];
    int ti[kTiMax];
    for (int i = 0; i < N; ++i) {
        xs[i] = s.px[e * N + i];
        ys[i] = s.py[e * N + i];
        ts[i] = s.pt[e * N + i];
    }
    for (int f = 0; f < nf; ++f) tf[f] = s.tf[static_cast<long long>(f) * B + e];
    for (int w = 0; w < ni; ++w) ti[w] = s.ti[static_cast<long long>(w) * B + e];
    int drones[MRSIM_MAX_ROBOTS];
    arctic_drones(c, drones);
    const EnvView<Real> v{xs, ys, ts, tf, ti, N, drones, nullptr};
    float* o = obs + e * N * D;
    for (int r = 0; r < N; ++r)
        for (int q = 0; q < D; ++q) o[r * D + q] = static_cast<float>(obs_feature<TASK, Real>(c, v, r, q, bdim));
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

// One trajectory record per (env, robot) of the state a step just wrote.
template <class Real>
__global__ void capture_kernel(DevState<Real> s, const int8_t* actions, const double* reward64, const uint8_t* done,
                               long long B, int N, mrsim_traj_record* out) {
    const long long t = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= B * N) return;
    const long long e = t / N;
    mrsim_traj_record rec;
    rec.x = double(s.px[t]);
    rec.y = double(s.py[t]);
    rec.theta = double(s.pt[t]);
    rec.reward = reward64[e];
    rec.metric = double(s.metric[e]);
    rec.collisions = s.collisions[e];
    rec.action = actions[t];
    rec.done = done[e];
    out[t] = rec;
}

}  // namespace mrsim_dev
