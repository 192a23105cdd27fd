// env_kernel.cuh — the fused step for small teams (N <= 4 robots, no rware
// obstacle rows): ONE THREAD PER ENVIRONMENT.
//
// The lane-per-robot step (step_kernel.cuh) spends most of its issue slots on
// group collectives (shuffles, votes, shared-memory publish/scan) that exist
// only to let 4 lanes cooperate on one 8-variable QP: ~5,000 lane-instructions
// per env-tick against ~500 algorithmic flops (ncu, profiles/r01_ncu_nav4_fp64.txt).
// Here a thread owns a whole env: the robots' poses, waypoints, sin/cos and
// the QP iterate live in registers with compile-time robot indices (NR = 4,
// runtime N <= 4 as predicates), nothing is exchanged between threads, and
// each thread's robot loops give 4-6 independent fp64 chains of ILP.
//
// Per step and env, the same pipeline as step_env (batch.hpp:165-224):
//   actions -> waypoints (framework.hpp:96-108, scenario.hpp:150-165)
//   sub_steps x [ hold rule / position or pose controller (controllers.hpp:34-92)
//                 -> CBF rows + dual active-set QP + map back (barrier.hpp:57-205, qp.hpp:183-357)
//                 -> unicycle Euler + wrap + arena clamp (core.hpp:102-118, batch.hpp:199-203)
//                 -> min pairwise distance / collision flag (batch.hpp:204-209) ]
//   -> transition / violation / step_index / done / finalize (batch.hpp:212-220)
//   -> observations (batch.hpp:143-151, 221) -> optional in-kernel auto-reset.
//
// QP: the method and discrete decisions of solve_qp (qp.hpp:183-357) with
// the inverse Gram matrix S = (N^T N)^-1 of the active normals kept up to
// date (bordered-inverse add, rank-1 downdate; see qp_group.cuh), run
// sequentially by the thread over its active list in the reference's order.
// Rows are scanned in the reference's order (pairs i<j, walls robot-major
// x-min/x-max/y-min/y-max, box sides per variable hi/lo; barrier.hpp:57-121,
// qp.hpp:104-141) with strict `v > worst`, so the first maximal row wins
// exactly as in the reference. The normalised pair rows of the tick live in
// shared memory, field-major [field][thread] (conflict-free, dynamically
// indexable); wall rows are recomputed from the projected points when
// scanned; the active-set workspace (<= 2N slots) is thread-local.
//
// Memory: the thread's N poses are 128-bit loads (double2 / float4) when N
// is 4; task fields are field-major [f][B] (coalesced across the warp);
// observations are staged per warp in shared memory and leave as one
// contiguous block of float4 stores (32 envs x N x D floats).
#pragma once

#include "step_kernel.cuh"

namespace mrsim_dev {

// Resident 64-thread blocks per SM the register budget is sized for: 7 x 64 x 148 SMs
// = 66,304 threads hold the 65,536-env benchmark batch in one wave (<= 144 registers).
#ifndef MRSIM_ENV_MINB
#define MRSIM_ENV_MINB 7
#endif

constexpr int kEnvNR = 4;           // robots per thread (compile-time bound)
constexpr int kEnvBlock = 64;       // threads (= envs) per block
constexpr int kEnvPairs = kEnvNR * (kEnvNR - 1) / 2;
constexpr int kEnvObsStageMax = 32 * 4 * 32;  // floats per warp of the obs stage (N*D <= 128)
// static shared memory of the kernel (fp64): pair rows, goal headings, waypoints, projected points
constexpr int kEnvStaticSmem = 8 * kEnvBlock * (3 * 6 + 4 + 8 + 8);

// Runtime index into a register array of NR values without local memory.
template <int NR, class T>
__device__ __forceinline__ T pick(const T (&a)[NR], int i) {
    T v = a[0];
#pragma unroll
    for (int k = 1; k < NR; ++k) v = (i == k) ? a[k] : v;
    return v;
}

// gamma * h^3 with the final product rounded on its own (never contracted into the
// caller's subtraction), so a wall row's rhs is the same value in the scan and in
// the QP step, as when it is stored (the lane-group kernel's row cache).
__device__ __forceinline__ double cube_rhs(double g, double h) { return __dmul_rn(g * h * h, h); }
__device__ __forceinline__ float cube_rhs(float g, float h) { return __fmul_rn(g * h * h, h); }

// Internal row ids (monotone in the reference's global row order for any N <= NR):
//   [0, 6)   pair slot s = (i, j), i < j < NR, lexicographic
//   [6, 22)  wall 4i + w of robot i (x-min, x-max, y-min, y-max)
//   [22, 38) box side 4i + b (x-hi, x-lo, y-hi, y-lo)
__device__ __forceinline__ int env_pi(int s) { return s < 3 ? 0 : (s < 5 ? 1 : 2); }
__device__ __forceinline__ int env_pj(int s) { return s == 0 ? 1 : (s == 1 ? 2 : (s == 2 ? 3 : (s == 3 ? 2 : 3))); }
constexpr int kRowWall = kEnvPairs;
constexpr int kRowBox = kEnvPairs + 4 * kEnvNR;
constexpr int kRowEnd = kRowBox + 4 * kEnvNR;

template <class Real>
struct TRow {  // +(cx, cy) on robot r1 and -(cx, cy) on r0 (pair), or (cx, cy) on r0 (r1 < 0); rhs h
    int r0, r1;
    Real cx, cy, h;
};

// Coefficient of a row on robot i (+1 / -1 / 0).
template <class Real>
__device__ __forceinline__ Real row_sign(const TRow<Real>& d, int i) {
    return (d.r1 >= 0) ? ((i == d.r1) ? Real(1) : ((i == d.r0) ? Real(-1) : Real(0)))
                       : ((i == d.r0) ? Real(1) : Real(0));
}
template <class Real>
__device__ __forceinline__ Real row_dot(const TRow<Real>& a, const TRow<Real>& b) {
    const Real sa0 = (a.r1 >= 0) ? Real(-1) : Real(1), sb0 = (b.r1 >= 0) ? Real(-1) : Real(1);
    const Real cc = a.cx * b.cx + a.cy * b.cy;
    Real s = 0;
    if (a.r0 == b.r0) s += sa0 * sb0 * cc;
    if (a.r0 == b.r1) s += sa0 * cc;
    if (a.r1 >= 0 && a.r1 == b.r0) s += sb0 * cc;
    if (a.r1 >= 0 && a.r1 == b.r1) s += cc;
    return s;
}

// One thread's barrier rows of the current tick.
template <class Real>
struct EnvRows {
    Real* rs;        // pair rows in shared memory: rs[(3s + f) * kEnvBlock], f = gx, gy, rhs
    const Real* pp;  // projected points in shared memory: pp[i * kEnvBlock] = x, pp[(NR + i) * kEnvBlock] = y
    int N, P;
    Real cap;
    const PhysConsts<Real>* k;

    __device__ __forceinline__ Real& F(int s, int f) const { return rs[(3 * s + f) * kEnvBlock]; }
    __device__ __forceinline__ Real px(int i) const { return pp[i * kEnvBlock]; }
    __device__ __forceinline__ Real py(int i) const { return pp[(kEnvNR + i) * kEnvBlock]; }
    __device__ __forceinline__ Real wall_h(int i, int w) const {
        return (w == 0) ? px(i) - k->wall_xmin
                        : (w == 1) ? k->wall_xmax - px(i) : (w == 2) ? py(i) - k->wall_ymin : k->wall_ymax - py(i);
    }
    __device__ __forceinline__ TRow<Real> describe(int id) const {
        TRow<Real> d;
        if (id < kRowWall) {
            d.r0 = env_pi(id);
            d.r1 = env_pj(id);
            d.cx = F(id, 0);
            d.cy = F(id, 1);
            d.h = F(id, 2);
        } else if (id < kRowBox) {
            const int q = id - kRowWall, w = q & 3;
            d.r0 = q >> 2;
            d.r1 = -1;
            d.cx = (w == 0) ? Real(-1) : ((w == 1) ? Real(1) : Real(0));
            d.cy = (w == 2) ? Real(-1) : ((w == 3) ? Real(1) : Real(0));
            d.h = cube_rhs(k->gamma, wall_h(d.r0, w));
        } else {
            const int q = id - kRowBox, b = q & 3;
            d.r0 = q >> 2;
            d.r1 = -1;
            d.cx = (b == 0) ? Real(1) : ((b == 1) ? Real(-1) : Real(0));
            d.cy = (b == 2) ? Real(1) : ((b == 3) ? Real(-1) : Real(0));
            d.h = cap;
        }
        return d;
    }
    // Most violated inactive row (qp.hpp:225-239): the first row (reference order) with the
    // largest violation above tol -- the reference's sequential strict `v > worst` scan.
    // The pair rows are reduced as a tree (independent chains; a right operand wins only when
    // strictly larger, so ties keep the lower index); the later wall and box rows are folded
    // in order, each robot's walls only when they can beat the current worst at all.
    __device__ __forceinline__ int scan(const Real (&ux)[kEnvNR], const Real (&uy)[kEnvNR], unsigned long long active,
                                        Real tol) const {
        Real pv[kEnvPairs];
#pragma unroll
        for (int s = 0; s < kEnvPairs; ++s) {
            const int i = s < 3 ? 0 : (s < 5 ? 1 : 2);
            const int j = s == 0 ? 1 : (s == 1 ? 2 : (s == 2 ? 3 : (s == 3 ? 2 : 3)));
            Real v = -Consts<Real>::inf;
            if (j < N && !((active >> s) & 1ull)) {
                const Real t = F(s, 0) * (ux[j] - ux[i]) + F(s, 1) * (uy[j] - uy[i]) - F(s, 2);
                if (t > tol) v = t;  // (NaN never qualifies, as in the sequential scan)
            }
            pv[s] = v;
        }
        // first-max tree over [tol, p0 .. p5]
        const bool b01 = pv[1] > pv[0], b23 = pv[3] > pv[2], b45 = pv[5] > pv[4];
        const Real v01 = b01 ? pv[1] : pv[0], v23 = b23 ? pv[3] : pv[2], v45 = b45 ? pv[5] : pv[4];
        const int i01 = b01 ? 1 : 0, i23 = b23 ? 3 : 2, i45 = b45 ? 5 : 4;
        const bool b03 = v23 > v01;
        const Real v03 = b03 ? v23 : v01;
        const int i03 = b03 ? i23 : i01;
        const bool b05 = v45 > v03;
        const Real vp = b05 ? v45 : v03;
        const int ip = b05 ? i45 : i03;
        Real worst = tol;
        int p = -1;
        if (vp > worst) {
            worst = vp;
            p = ip;
        }
#pragma unroll
        for (int i = 0; i < kEnvNR; ++i) {
            const Real h0 = px(i) - k->wall_xmin, h1 = k->wall_xmax - px(i);
            const Real h2 = py(i) - k->wall_ymin, h3 = k->wall_ymax - py(i);
            // Exact skip of the robot's four wall rows: the rounded cube is monotone, so every
            // v_w = fl(+-u - cube(h_w)) <= fl(max|u| - cube(min h)); if that bound does not beat
            // `worst`, no wall row of this robot can (the strict `v > worst` test).
            const Real bound = dmax(dabs(ux[i]), dabs(uy[i])) - cube_rhs(k->gamma, dmin(dmin(h0, h1), dmin(h2, h3)));
            if (i < N && bound > worst) {
                const int w0 = kRowWall + 4 * i;
                Real v;
                v = -ux[i] - cube_rhs(k->gamma, h0);
                if (!((active >> (w0 + 0)) & 1ull) && v > worst) { worst = v; p = w0 + 0; }
                v = ux[i] - cube_rhs(k->gamma, h1);
                if (!((active >> (w0 + 1)) & 1ull) && v > worst) { worst = v; p = w0 + 1; }
                v = -uy[i] - cube_rhs(k->gamma, h2);
                if (!((active >> (w0 + 2)) & 1ull) && v > worst) { worst = v; p = w0 + 2; }
                v = uy[i] - cube_rhs(k->gamma, h3);
                if (!((active >> (w0 + 3)) & 1ull) && v > worst) { worst = v; p = w0 + 3; }
            }
        }
        // box sides (fold_rows qp.hpp:126-139): a side can only be violated beyond tol when |u| > cap
#pragma unroll
        for (int i = 0; i < kEnvNR; ++i) {
            if (i < N && (dabs(ux[i]) > cap || dabs(uy[i]) > cap)) {
                const int b0 = kRowBox + 4 * i;
                Real v;
                v = ux[i] - cap;
                if (!((active >> (b0 + 0)) & 1ull) && v > worst) { worst = v; p = b0 + 0; }
                v = -ux[i] - cap;
                if (!((active >> (b0 + 1)) & 1ull) && v > worst) { worst = v; p = b0 + 1; }
                v = uy[i] - cap;
                if (!((active >> (b0 + 2)) & 1ull) && v > worst) { worst = v; p = b0 + 2; }
                v = -uy[i] - cap;
                if (!((active >> (b0 + 3)) & 1ull) && v > worst) { worst = v; p = b0 + 3; }
            }
        }
        return p;
    }
};

// The CBF QP of one env (solve_qp, qp.hpp:183-357) for 2N <= 8 variables held
// in registers. Returns kQpOptimal / kQpInfeasible / kQpIterLimit.
// p0: the most violated row at u_nom (the caller's first scan, >= 0).
template <class Real>
__device__ __forceinline__ int env_qp_solve(const EnvRows<Real>& rows, Real (&ux)[kEnvNR], Real (&uy)[kEnvNR],
                                            int total_rows, Real tol, int p0) {
    constexpr int K = 2 * kEnvNR;  // max active rows (independent normals in R^{2N})
    Real S[K * K];                 // inverse Gram of the active normals, logical order
    Real lam[K], rv[K];
    TRow<Real> act[K];
    int act_id[K];
    int k = 0;
    unsigned long long active = 0;
    const int max_iterations = 100 + 20 * total_rows;  // qp.hpp:193
    int status = kQpOptimal;
    for (int iter = 0;; ++iter) {
        if (iter >= max_iterations) {
            status = kQpIterLimit;
            break;
        }
        const int p = iter == 0 ? p0 : rows.scan(ux, uy, active, tol);
        if (p < 0) break;
        const TRow<Real> g = rows.describe(p);
        const Real gn = (g.r1 >= 0 ? Real(2) : Real(1)) * (g.cx * g.cx + g.cy * g.cy);
        if (gn < Prec<Real>::eps_row) {  // zero-norm violated row (qp.hpp:242-253)
            status = kQpInfeasible;
            break;
        }
        bool added = false;
        Real lam_p = 0;
        for (int guard = 0; guard <= total_rows && !added; ++guard) {  // qp.hpp:262-330
            // r = S N^T g
            Real d[K];
            for (int a = 0; a < k; ++a) d[a] = row_dot(act[a], g);
            for (int a = 0; a < k; ++a) {
                Real s = 0;
                for (int c = 0; c < k; ++c) s += S[a * K + c] * d[c];
                rv[a] = s;
            }
            // z = g - N r (dense over the robots; the rows touch <= 2 of them)
            Real zx[kEnvNR], zy[kEnvNR];
#pragma unroll
            for (int i = 0; i < kEnvNR; ++i) {
                const Real sg = row_sign(g, i);
                zx[i] = sg * g.cx;
                zy[i] = sg * g.cy;
            }
            for (int a = 0; a < k; ++a) {
#pragma unroll
                for (int i = 0; i < kEnvNR; ++i) {
                    const Real sa = row_sign(act[a], i);
                    zx[i] -= rv[a] * (sa * act[a].cx);
                    zy[i] -= rv[a] * (sa * act[a].cy);
                }
            }
            Real z2 = 0, gu = 0;
#pragma unroll
            for (int i = 0; i < kEnvNR; ++i) {
                if (i < rows.N) {
                    z2 += zx[i] * zx[i] + zy[i] * zy[i];
                    const Real sg = row_sign(g, i);
                    gu += (sg * g.cx) * ux[i] + (sg * g.cy) * uy[i];
                }
            }
            const Real viol = gu - g.h;  // qp.hpp:281
            if (viol <= tol) {            // qp.hpp:282-289
                if (lam_p > Real(0) && z2 > Prec<Real>::eps_z) {
                    // bordered inverse: the new slot's Schur complement is |z|^2
                    const Real is = Real(1) / z2;
                    for (int a = 0; a < k; ++a) {
                        const Real ra = rv[a] * is;
                        for (int c = 0; c < k; ++c) S[a * K + c] += ra * rv[c];
                        S[a * K + k] = -ra;
                        S[k * K + a] = -ra;
                    }
                    S[k * K + k] = is;
                    act[k] = g;
                    act_id[k] = p;
                    lam[k] = lam_p;
                    active |= 1ull << p;
                    ++k;
                }
                added = true;
                break;
            }
            // first blocking multiplier in active-list order (qp.hpp:291-302)
            Real t1 = Consts<Real>::inf;
            int bi = -1;
            for (int a = 0; a < k; ++a) {
                if (rv[a] > Prec<Real>::eps_r) {
                    const Real t = lam[a] / rv[a];
                    if (t < t1) {
                        t1 = t;
                        bi = a;
                    }
                }
            }
            bool drop = false, add = false;
            if (z2 <= Prec<Real>::eps_z) {  // qp.hpp:304-315
                if (bi < 0) {
                    status = kQpInfeasible;
                    return status;
                }
                for (int a = 0; a < k; ++a) lam[a] -= t1 * rv[a];
                lam_p += t1;
                drop = true;
            } else {  // qp.hpp:317-329
                const Real t2 = viol / z2;
                const Real t = dmin(t1, t2);
#pragma unroll
                for (int i = 0; i < kEnvNR; ++i) {
                    ux[i] -= t * zx[i];
                    uy[i] -= t * zy[i];
                }
                for (int a = 0; a < k; ++a) lam[a] -= t * rv[a];
                lam_p += t;
                if (t2 <= t1) add = true;
                else drop = true;
            }
            if (add) {
                const Real is = Real(1) / z2;
                for (int a = 0; a < k; ++a) {
                    const Real ra = rv[a] * is;
                    for (int c = 0; c < k; ++c) S[a * K + c] += ra * rv[c];
                    S[a * K + k] = -ra;
                    S[k * K + a] = -ra;
                }
                S[k * K + k] = is;
                act[k] = g;
                act_id[k] = p;
                lam[k] = lam_p;
                active |= 1ull << p;
                ++k;
                added = true;
            }
            if (drop) {  // S <- S_{-b,-b} - S_{-b,b} S_{b,-b} / S_bb, then close the gap
                const Real ib = Real(1) / S[bi * K + bi];
                for (int a = 0; a < k; ++a) {
                    if (a == bi) continue;
                    const Real sab = S[a * K + bi] * ib;
                    for (int c = 0; c < k; ++c)
                        if (c != bi) S[a * K + c] -= sab * S[bi * K + c];
                }
                active &= ~(1ull << act_id[bi]);
                for (int a = bi; a + 1 < k; ++a) {
                    act[a] = act[a + 1];
                    act_id[a] = act_id[a + 1];
                    lam[a] = lam[a + 1];
                }
                for (int a = 0; a < k; ++a)
                    for (int c = bi; c + 1 < k; ++c) S[a * K + c] = S[a * K + c + 1];
                for (int a = bi; a + 1 < k; ++a)
                    for (int c = 0; c + 1 < k; ++c) S[a * K + c] = S[(a + 1) * K + c];
                --k;
            }
        }
        if (!added) break;  // stall (qp.hpp:331-334)
    }
    return status;
}

// The QP iterate in and out of env_qp (by value: the rare QP path is an out-of-line
// call, so the common tick -- nothing violated at u_nom -- keeps its registers).
template <class Real>
struct QpIO {
    Real ux[kEnvNR], uy[kEnvNR];
    int status;
};

template <class Real>
__device__ __noinline__ QpIO<Real> env_qp(const EnvRows<Real> rows, QpIO<Real> io, int total_rows, Real tol, int p0) {
    Real(&ux)[kEnvNR] = io.ux;
    Real(&uy)[kEnvNR] = io.uy;
    io.status = env_qp_solve<Real>(rows, ux, uy, total_rows, tol, p0);
    return io;
}

template <class Real, int TASK>
__global__ void __launch_bounds__(kEnvBlock, MRSIM_ENV_MINB) env_step_kernel(const __grid_constant__ StepParams<Real> p) {
    constexpr int NR = kEnvNR;
    if (*p.err != ~0ull) return;  // sticky device error: later steps are no-ops
    __shared__ Real pair_rows[3 * kEnvPairs * kEnvBlock];
    __shared__ Real goal_heading[kEnvNR * kEnvBlock];  // pose controller: the step's goal headings [robot][thread]
    __shared__ Real waypoint[2 * kEnvNR * kEnvBlock];  // the step's waypoints [x: robot | y: robot][thread]
    __shared__ Real proj_pt[2 * kEnvNR * kEnvBlock];   // the tick's projected points, same layout
    extern __shared__ __align__(16) float env_obs_stage[];  // [warps][32 * N * D] when p.obs_stage

    const mrsim_cfg& c = p.c;
    const int N = p.N;
    const PhysConsts<Real>& K = p.k;
    const long long e_real = p.e_begin + static_cast<long long>(blockIdx.x) * kEnvBlock + threadIdx.x;
    const bool ghost = e_real >= p.e_end;
    const long long e = ghost ? p.e_end - 1 : e_real;

    // ---- load ----
    const int step_index = p.in.step_index[e];
    const uint64_t key = p.in.key[e];
    Real x[NR], y[NR], th[NR];
    if (N == NR && sizeof(Real) == 8) {  // 2 x 128-bit per field
        const double2* px = reinterpret_cast<const double2*>(p.in.px + e * NR);
        const double2* py = reinterpret_cast<const double2*>(p.in.py + e * NR);
        const double2* pt = reinterpret_cast<const double2*>(p.in.pt + e * NR);
        const double2 a0 = px[0], a1 = px[1], b0 = py[0], b1 = py[1], c0 = pt[0], c1 = pt[1];
        x[0] = a0.x; x[1] = a0.y; x[2] = a1.x; x[3] = a1.y;
        y[0] = b0.x; y[1] = b0.y; y[2] = b1.x; y[3] = b1.y;
        th[0] = c0.x; th[1] = c0.y; th[2] = c1.x; th[3] = c1.y;
    } else if (N == NR) {  // fp32: one 128-bit load per field
        const float4 a = *reinterpret_cast<const float4*>(p.in.px + e * NR);
        const float4 b = *reinterpret_cast<const float4*>(p.in.py + e * NR);
        const float4 t = *reinterpret_cast<const float4*>(p.in.pt + e * NR);
        x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
        y[0] = b.x; y[1] = b.y; y[2] = b.z; y[3] = b.w;
        th[0] = t.x; th[1] = t.y; th[2] = t.z; th[3] = t.w;
    } else {
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            x[i] = i < N ? p.in.px[e * N + i] : Real(0);
            y[i] = i < N ? p.in.py[e * N + i] : Real(0);
            th[i] = i < N ? p.in.pt[e * N + i] : Real(0);
        }
    }
    Real tf[kTfMax];
    int ti[kTiMax];
    for (int f = 0; f < p.nf; ++f) tf[f] = p.in.tf[static_cast<long long>(f) * p.B + e];
    for (int w = 0; w < p.ni; ++w) ti[w] = p.in.ti[static_cast<long long>(w) * p.B + e];

    // ---- actions (validate_actions, batch.hpp:226-237) ----
    int act[NR];
    int bad_robot = -1, bad_act = 0;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        act[i] = 0;
        if (i < N) {
            act[i] = p.actions ? static_cast<int>(p.actions[e * N + i])
                               : (p.actions32 ? p.actions32[e * N + i] : policy_action(p.in.pkey[e], step_index, i));
            if (bad_robot < 0 && (act[i] < 0 || act[i] >= 5)) {
                bad_robot = i;
                bad_act = act[i];
            }
        }
    }
    if (bad_robot >= 0 && !ghost) {
        report_error(p.err, e, bad_robot, kErrInvalidAction, bad_act);
        *p.err_serial = p.serial;
    }
    bool skip = ghost || bad_robot >= 0;  // compute, never store

    // ---- waypoints (Scenario::waypoints + action_to_waypoint) ----
    const uint64_t skey = fork_key(key, 1ull + static_cast<uint64_t>(step_index));  // step_stream
    Real* wth = goal_heading + threadIdx.x;  // wth[i * kEnvBlock]
    Real* wps = waypoint + threadIdx.x;      // x of robot i at [i * kEnvBlock], y at [(NR + i) * kEnvBlock]
    Real* pps = proj_pt + threadIdx.x;
    const bool pose_ctl = c.controller == MRSIM_CONTROLLER_UNICYCLE_POSE;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        Real wx = x[i], wy = y[i];
        if (i < N) {
            if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {  // actions ignored: the stored targets (random_waypoints.hpp:40-44)
                wx = tf[2 * i];
                wy = tf[2 * i + 1];
            } else {
                const Real ss = step_size_of<TASK, Real>(c, ti, i, x[i], y[i]);
                const Real dxa = (act[i] == 3) ? Real(-1) : ((act[i] == 4) ? Real(1) : Real(0));
                const Real dya = (act[i] == 1) ? Real(1) : ((act[i] == 2) ? Real(-1) : Real(0));
                wx = x[i] + dxa * ss;
                wy = y[i] + dya * ss;
                if (c.action_noise_scale > 0.0) {
                    const double half = c.action_noise_scale * static_cast<double>(ss);
                    Rng nr{skey, static_cast<uint64_t>(2 * i)};
                    wx += static_cast<Real>(nr.uniform(-half, half));
                    wy += static_cast<Real>(nr.uniform(-half, half));
                }
                wx = dclamp(wx, -K.hw, K.hw);
                wy = dclamp(wy, -K.hh, K.hh);
            }
        }
        wps[i * kEnvBlock] = wx;
        wps[(NR + i) * kEnvBlock] = wy;
    }
    // goal headings for the pose controller (Scenario::waypoint_headings, batch.hpp:169-171)
    if (pose_ctl) {
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            Real h = th[i];
            if (i < N) {
                if (TASK == MRSIM_TASK_RANDOM_WAYPOINTS) {
                    h = tf[2 * N + i];  // random_waypoints.hpp:46-50
                } else {  // scenario.hpp:168-177
                    const Real ddx = wps[i * kEnvBlock] - x[i], ddy = wps[(NR + i) * kEnvBlock] - y[i];
                    h = dhypot(ddx, ddy) > Real(1e-12) ? atan2(ddy, ddx) : th[i];
                }
            }
            wth[i * kEnvBlock] = h;
        }
    }

    // ---- physics ticks ----
    const int P = N * (N - 1) / 2;
    const int total_rows = P + 4 * N + 4 * N;
    EnvRows<Real> rows;
    rows.rs = pair_rows + threadIdx.x;
    rows.pp = pps;
    rows.N = N;
    rows.P = P;
    rows.cap = K.cap;
    rows.k = &K;
    Real min_dist = p.in.min_dist[e];
    Real min_d2 = Consts<Real>::inf;
    int qp_inf = p.in.qp_inf[e];
    bool collision = false;
    for (int tick = 0; tick < c.sub_steps; ++tick) {
        Real sn[NR], cs[NR], nv[NR], nw[NR], prx[NR], pry[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            dsincos(th[i], &sn[i], &cs[i]);
            prx[i] = x[i] + cs[i] * K.l;  // projected_point (controllers.hpp:34-36)
            pry[i] = y[i] + sn[i] * K.l;
            pps[i * kEnvBlock] = prx[i];
            pps[(NR + i) * kEnvBlock] = pry[i];
            nv[i] = 0;
            nw[i] = 0;
            const Real wx = wps[i * kEnvBlock], wy = wps[(NR + i) * kEnvBlock];
            if (pose_ctl) {  // unicycle_pose_controller (controllers.hpp:68-82), out of line
                const Real2<Real> c2 = pose_nominal<Real>(K, x[i], y[i], th[i], wx, wy, wth[i * kEnvBlock]);
                nv[i] = c2.a;
                nw[i] = c2.b;
            } else if (!(wx == x[i] && wy == y[i])) {  // hold rule (batch.hpp:187-188)
                Real ux = K.k_pos * (wx - prx[i]);
                Real uy = K.k_pos * (wy - pry[i]);
                const Real nrm = dsqrt(ux * ux + uy * uy);
                if (!(nrm <= K.si_max || nrm == Real(0))) {
                    const Real sc = K.si_max / nrm;
                    ux *= sc;
                    uy *= sc;
                }
                nv[i] = dclamp(cs[i] * ux + sn[i] * uy, -K.v_max, K.v_max);
                nw[i] = dclamp((-sn[i] * ux + cs[i] * uy) * K.inv_l, -K.w_max, K.w_max);
            }
        }
        Real cv[NR], cw[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            cv[i] = nv[i];
            cw[i] = nw[i];
        }
        if (c.barrier_enabled) {  // apply_barrier (barrier.hpp:132-205)
            Real ux[NR], uy[NR];
#pragma unroll
            for (int i = 0; i < NR; ++i) {  // u_nom = uni_to_si(clamped nominal) (controllers.hpp:59-65)
                ux[i] = i < N ? cs[i] * nv[i] - K.l * sn[i] * nw[i] : Real(0);
                uy[i] = i < N ? sn[i] * nv[i] + K.l * cs[i] * nw[i] : Real(0);
            }
            // pair rows at the projected points (barrier.hpp:69-83 + fold_rows qp.hpp:104-125)
            bool coincident = false;
#pragma unroll
            for (int s = 0; s < kEnvPairs; ++s) {
                const int i = s < 3 ? 0 : (s < 5 ? 1 : 2);
                const int j = s == 0 ? 1 : (s == 1 ? 2 : (s == 2 ? 3 : (s == 3 ? 2 : 3)));
                if (j < N) {
                    const Real dx = prx[i] - prx[j], dy = pry[i] - pry[j];
                    const Real dist2 = dx * dx + dy * dy;
                    if (dist2 < Real(1e-18)) coincident = true;
                    const Real h = dist2 - K.r_eff2;
                    const Real inv = rsqrt(Real(8) * dist2);
                    rows.F(s, 0) = Real(2) * dx * inv;
                    rows.F(s, 1) = Real(2) * dy * inv;
                    rows.F(s, 2) = K.gamma * h * h * h * inv;
                }
            }
            int status = kQpOptimal;
            if (coincident) {
                if (!skip) {
                    report_error(p.err, e, 0, kErrCoincident);
                    *p.err_serial = p.serial;
                }
                skip = true;
            } else {
                const int p0 = rows.scan(ux, uy, 0ull, K.tol);  // most ticks: nothing violated at u_nom
                if (p0 >= 0) {
                    QpIO<Real> io;
#pragma unroll
                    for (int i = 0; i < NR; ++i) {
                        io.ux[i] = ux[i];
                        io.uy[i] = uy[i];
                    }
                    io = env_qp<Real>(rows, io, total_rows, K.tol, p0);
#pragma unroll
                    for (int i = 0; i < NR; ++i) {
                        ux[i] = io.ux[i];
                        uy[i] = io.uy[i];
                    }
                    status = io.status;
                }
            }
            // map back + uniform scale (barrier.hpp:186-204)
            Real scale = 1;
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                cv[i] = cs[i] * ux[i] + sn[i] * uy[i];
                cw[i] = (-sn[i] * ux[i] + cs[i] * uy[i]) * K.inv_l;
                if (i < N) {
                    if (dabs(cv[i]) > K.v_max) scale = dmin(scale, K.v_max / dabs(cv[i]));
                    if (dabs(cw[i]) > K.w_max) scale = dmin(scale, K.w_max / dabs(cw[i]));
                }
            }
            const bool zero = status == kQpInfeasible;  // barrier.hpp:178-182
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                cv[i] = zero ? Real(0) : cv[i] * scale;
                cw[i] = zero ? Real(0) : cw[i] * scale;
            }
            if (status == kQpInfeasible) ++qp_inf;
        }
        // unicycle Euler step + wrap + arena clamp (core.hpp:112-118, batch.hpp:199-203)
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            x[i] = x[i] + cv[i] * cs[i] * K.dt;
            y[i] = y[i] + cv[i] * sn[i] * K.dt;
            const Real tn = th[i] + cw[i] * K.dt;
            if (i < N && !skip && !isfinite(tn)) {
                report_error(p.err, e, i, kErrNonFinite);
                *p.err_serial = p.serial;
            }
            th[i] = wrap_angle_dev(tn);
            x[i] = dclamp(x[i], -K.hw, K.hw);
            y[i] = dclamp(y[i], -K.hh, K.hh);
        }
        // collision check (batch.hpp:204-209); sqrt is monotone, so it is taken once per step
        if (N > 1) {
            Real md2 = Consts<Real>::inf;
#pragma unroll
            for (int s = 0; s < kEnvPairs; ++s) {
                const int i = s < 3 ? 0 : (s < 5 ? 1 : 2);
                const int j = s == 0 ? 1 : (s == 1 ? 2 : (s == 2 ? 3 : (s == 3 ? 2 : 3)));
                if (j < N) {
                    const Real dx = x[i] - x[j], dy = y[i] - y[j];
                    md2 = dmin(md2, dx * dx + dy * dy);
                }
            }
            min_d2 = dmin(min_d2, md2);
            collision = collision || md2 < K.coll_r2;
        }
    }
    min_dist = dmin(min_dist, dsqrt(min_d2));

    // ---- transition, bookkeeping (batch.hpp:212-220) ----
    Real xs[NR], ys[NR], ts[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
        xs[i] = x[i];
        ys[i] = y[i];
        ts[i] = th[i];
    }
    int drones[NR];
    if (TASK == MRSIM_TASK_ARCTIC_TRANSPORT) arctic_drones(c, drones);
    EnvView<Real> view{xs, ys, ts, tf, ti, N, drones, p.prey_off, nullptr, nullptr};
    Real metric = p.in.metric[e];
    int success = p.in.success[e];
    int collisions = p.in.collisions[e];
    Real ep_return = p.in.ep_return[e];
    // the transition continues the step stream after the waypoint noise draws
    Rng trng{skey, (c.action_noise_scale > 0.0 && TASK != MRSIM_TASK_RANDOM_WAYPOINTS) ? static_cast<uint64_t>(2 * N)
                                                                                        : 0ull};
    Real reward = transition_task<TASK, Real>(c, view, trng, metric);
    if (collision) {
        collisions += 1;
        reward += Real(c.coef[MRSIM_COEF_VIOLATION]);
    }
    const int new_step = step_index + 1;
    const int done = new_step >= c.max_steps ? 1 : 0;
    if (done) finalize_task<TASK, Real>(c, view, metric, success);
    ep_return += reward;
    if (!skip) {
        if (p.reward) p.reward[e] = static_cast<float>(reward);
        if (p.reward64) p.reward64[e] = static_cast<double>(reward);
        if (p.done) p.done[e] = static_cast<uint8_t>(done);
        if (done && new_step == c.max_steps)  // EpisodeStats (harness.hpp:277-285)
            stats_commit(p.st, e, p.serial, static_cast<double>(ep_return), static_cast<double>(metric), success,
                         collisions, qp_inf, static_cast<double>(min_dist));
    }

    // ---- observations (assemble_observations, batch.hpp:143-151) ----
    const int ND = N * p.D;
    if (p.obs) {
        if (p.obs_stage) {
            // the warp's 32 envs are consecutive: stage their obs, then one contiguous block of float4 stores
            const int lane = threadIdx.x & 31;
            float* wst = env_obs_stage + (threadIdx.x >> 5) * p.obs_stage;
            float* mine = wst + lane * ND;
            for (int r = 0; r < N; ++r)
                for (int q = 0; q < p.D; ++q)
                    mine[r * p.D + q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, q, p.bdim));
            __syncwarp();
            const long long e0 = e_real - lane;
            const long long left = p.e_end - e0;
            const int total = static_cast<int>(left < 32 ? left : 32) * ND;
            float* dst = p.obs + e0 * ND;
            if (((e0 * ND) & 3) == 0 && (total & 3) == 0) {
                const float4* src4 = reinterpret_cast<const float4*>(wst);
                float4* dst4 = reinterpret_cast<float4*>(dst);
                for (int k = lane; k < total / 4; k += 32) dst4[k] = src4[k];
            } else {
                for (int k = lane; k < total; k += 32) dst[k] = wst[k];
            }
            __syncwarp();
        } else if (!skip) {
            float* o = p.obs + e * ND;
            for (int r = 0; r < N; ++r)
                for (int q = 0; q < p.D; ++q)
                    o[r * p.D + q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, q, p.bdim));
        }
    }

    uint64_t okey = key, oseed = p.in.seed[e], opkey = p.in.pkey[e];
    long long oepisode = p.in.episode[e];
    int ostep = new_step;
    // ---- auto-reset (harness wave semantics, harness.hpp:227-232) ----
    if (p.auto_reset && done && !skip) {
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
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            xs[i] = i < N ? static_cast<Real>(ro.x[i]) : Real(0);
            ys[i] = i < N ? static_cast<Real>(ro.y[i]) : Real(0);
            ts[i] = i < N ? static_cast<Real>(ro.th[i]) : Real(0);
        }
        for (int f = 0; f < p.nf; ++f) tf[f] = static_cast<Real>(ro.tf[f]);
        for (int w = 0; w < p.ni; ++w) ti[w] = ro.ti[w];
        ostep = 0;
        collisions = 0;
        qp_inf = 0;
        success = 0;
        metric = 0;
        min_dist = Consts<Real>::inf;
        ep_return = 0;
        okey = nkey;
        oseed = seed;
        opkey = policy_key_of(seed);
        oepisode = episode;
        if (p.next_obs) {
            float* o = p.next_obs + e * ND;
            for (int r = 0; r < N; ++r)
                for (int q = 0; q < p.D; ++q)
                    o[r * p.D + q] = static_cast<float>(obs_feature<TASK, Real>(c, view, r, q, p.bdim));
        }
    }

    // ---- store ----
    if (skip) return;
    if (N == NR && sizeof(Real) == 8) {
        double2* px = reinterpret_cast<double2*>(p.out.px + e * NR);
        double2* py = reinterpret_cast<double2*>(p.out.py + e * NR);
        double2* pt = reinterpret_cast<double2*>(p.out.pt + e * NR);
        px[0] = make_double2(xs[0], xs[1]);
        px[1] = make_double2(xs[2], xs[3]);
        py[0] = make_double2(ys[0], ys[1]);
        py[1] = make_double2(ys[2], ys[3]);
        pt[0] = make_double2(ts[0], ts[1]);
        pt[1] = make_double2(ts[2], ts[3]);
    } else if (N == NR) {
        *reinterpret_cast<float4*>(p.out.px + e * NR) = make_float4(xs[0], xs[1], xs[2], xs[3]);
        *reinterpret_cast<float4*>(p.out.py + e * NR) = make_float4(ys[0], ys[1], ys[2], ys[3]);
        *reinterpret_cast<float4*>(p.out.pt + e * NR) = make_float4(ts[0], ts[1], ts[2], ts[3]);
    } else {
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            if (i < N) {
                p.out.px[e * N + i] = xs[i];
                p.out.py[e * N + i] = ys[i];
                p.out.pt[e * N + i] = ts[i];
            }
        }
    }
    for (int f = 0; f < p.nf; ++f) p.out.tf[static_cast<long long>(f) * p.B + e] = tf[f];
    for (int w = 0; w < p.ni; ++w) p.out.ti[static_cast<long long>(w) * p.B + e] = ti[w];
    p.out.step_index[e] = ostep;
    p.out.collisions[e] = collisions;
    p.out.qp_inf[e] = qp_inf;
    p.out.success[e] = success;
    p.out.metric[e] = metric;
    p.out.min_dist[e] = min_dist;
    p.out.ep_return[e] = ep_return;
    p.out.key[e] = okey;
    p.out.seed[e] = oseed;
    p.out.pkey[e] = opkey;
    p.out.episode[e] = oepisode;
}

}  // namespace mrsim_dev
