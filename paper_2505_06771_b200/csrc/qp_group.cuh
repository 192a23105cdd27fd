// qp_group.cuh — the CBF safety QP, solved cooperatively by the L lanes of
// one environment group, in warp lockstep (see group.cuh).
//
//   minimize 0.5 ||u - u_nom||^2   s.t.  g_r . u <= h_r   (unit-norm rows)
//
// Same algorithm and the same discrete decisions as the reference's
// solve_qp (qp.hpp:183-357): Goldfarb-Idnani dual active set with H = I,
// most-violated row first (ties -> lowest row index), partial dual steps
// that drop the first blocking multiplier, infeasibility when the entering
// normal is dependent and nothing blocks. B200-native differences:
//   * the active set is kept as an incrementally updated QR factorisation
//     N = Q R (Q: n x k orthonormal columns, R: k x k upper triangular) in
//     shared memory, instead of re-forming and re-factorising the Gram
//     matrix N^T N at every inner step (qp.hpp:199-221). Adding a row is one
//     Gram-Schmidt column (the residual z the step needs anyway), dropping
//     a row is k Givens rotations; r = (N^T N)^{-1} N^T g = R^{-1} Q^T g.
//   * lane l owns variables 2l, 2l+1 (one robot: u_x, u_y) and active slots
//     l, l+L, ...; reductions are shuffles over the group's lanes.
//   * every loop that contains a collective has a warp-uniform trip count;
//     per-environment decisions are predicates, so the whole warp (32/L
//     environments) runs in lockstep with full-mask shuffles.
//   * rows are never materialised: the RowSet policy evaluates them on the
//     fly (barrier rows from the robots' projected points, or dense rows
//     for the unit-level entry point).
#pragma once

#include "group.cuh"
#include "mrsim_device.cuh"

namespace mrsim_dev {

enum QpStatusDev : int { kQpOptimal = 0, kQpInfeasible = 1, kQpIterLimit = 2 };

// Shared-memory workspace of one group for n variables:
//   Q[a*n + v] (column a = active slot a), R[col*n + row] (upper triangular),
//   Rd[a] = 1 / R[a][a], gS (entering normal), cS (Q^T g).
// Per-slot scalars (c_a, r_a, lambda_a, row id) live in registers of lane
// a % L (slots a = lane and a = lane + L; k <= n = 2N <= 2L).
template <class Real>
struct QpWs {
    Real *Q, *R, *Rd, *gS, *cS;
    static __host__ __device__ constexpr int reals(int n) { return 2 * n * n + 3 * n; }
    static __host__ __device__ constexpr int ints(int) { return 0; }
    __device__ void carve(Real* base, int*, int n) {
        Q = base;
        R = Q + n * n;
        Rd = R + n * n;
        gS = Rd + n;
        cS = gS + n;
    }
};

// Slot registers of one lane: slots a0 = lane, a1 = lane + L.
template <class Real>
struct Slots {
    Real c0, c1, r0, r1, lam0, lam1;
    int act0, act1;
};

// Drop active slot `bi` of the groups with do_drop set (the reference erases
// active[b] / lambda[b] and re-factorises, qp.hpp:270-271, 312-313, 327-328):
// delete column bi of R and restore triangularity with Givens rotations that
// are applied to Q's columns as well. Order of the remaining slots is kept.
template <class Real, int L, class RowSet>
__device__ __forceinline__ void qp_drop(const Grp<L>& g, RowSet& rows, const QpWs<Real>& ws, Slots<Real>& sl, int n,
                                        int& k, bool do_drop, int bi) {
    const int lane = g.lane;
    const int a0 = lane, a1 = lane + L;
    // clear the dropped row's active bit (row id lives on lane bi % L)
    const int bsrc = bi < 0 ? 0 : (bi & (L - 1));
    const int dr0 = g.shfl(sl.act0, bsrc), dr1 = g.shfl(sl.act1, bsrc);  // both unconditionally (lockstep)
    const int drop_row = (bi >= L) ? dr1 : dr0;
    if (do_drop) rows.set_active(g, drop_row, false);
    // shift slots (bi, k) down by one: slot a takes slot a+1
    const int nxt = (lane + 1) & (L - 1);
    const Real l0n = g.shfl(sl.lam0, nxt), l1n = g.shfl(sl.lam1, nxt);
    const int c0n = g.shfl(sl.act0, nxt), c1n = g.shfl(sl.act1, nxt);
    const Real l1_from0 = g.shfl(sl.lam1, 0);
    const int c1_from0 = g.shfl(sl.act1, 0);
    if (do_drop) {
        if (a0 >= bi && a0 < k - 1) {
            sl.lam0 = (lane < L - 1) ? l0n : l1_from0;
            sl.act0 = (lane < L - 1) ? c0n : c1_from0;
        }
        if (a1 >= bi && a1 < k - 1) {
            sl.lam1 = l1n;
            sl.act1 = c1n;
        }
        // delete column bi of R (this lane's rows)
        for (int row = lane; row < k; row += L)
            for (int col = bi; col < k - 1; ++col) ws.R[col * n + row] = ws.R[(col + 1) * n + row];
    }
    Grp<L>::sync();
    const int jmax = Grp<L>::warp_max(do_drop ? k - 1 : 0);
    for (int j = 0; j < jmax; ++j) {
        const bool rot = do_drop && j >= bi && j < k - 1;
        Real a = 0, bb = 0;
        if (rot) {
            a = ws.R[j * n + j];
            bb = ws.R[j * n + j + 1];
        }
        Grp<L>::sync();
        if (rot) {
            const Real rho = dsqrt(a * a + bb * bb);
            const Real cg = a / rho, sg = bb / rho;
            for (int col = lane; col < k - 1; col += L) {
                if (col < j) continue;
                const Real x = ws.R[col * n + j], y = ws.R[col * n + j + 1];
                ws.R[col * n + j] = cg * x + sg * y;
                ws.R[col * n + j + 1] = (col == j) ? Real(0) : (-sg * x + cg * y);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int v = 2 * lane + h;
                if (v >= n) continue;
                const Real x = ws.Q[j * n + v], y = ws.Q[(j + 1) * n + v];
                ws.Q[j * n + v] = cg * x + sg * y;
                ws.Q[(j + 1) * n + v] = -sg * x + cg * y;
            }
        }
        Grp<L>::sync();
    }
    if (do_drop) {
        --k;
        for (int a = lane; a < k; a += L)
            if (a >= bi) ws.Rd[a] = Real(1) / ws.R[a * n + a];
    }
}

// Solve for the groups with `participate` set. (ux, uy): this lane's pair of
// variables (in: u_nom, out: solution). Returns the QpStatusDev of the group.
template <class Real, int L, class RowSet>
__device__ __forceinline__ int qp_solve(const Grp<L>& g, RowSet& rows, const QpWs<Real>& ws, int n, bool participate, Real& ux,
                        Real& uy, int total_rows, Real tol) {
    const int lane = g.lane;
    const bool vl = 2 * lane < n;      // this lane's x variable exists
    const bool vly = 2 * lane + 1 < n;  // ... and its y variable (n may be odd for dense QPs)
    const int a0 = lane, a1 = lane + L;
    Slots<Real> sl{0, 0, 0, 0, 0, 0, 0, 0};
    int k = 0;
    int status = kQpOptimal;
    bool done = !participate;
    int iter = 0;
    const int max_iterations = 100 + 20 * total_rows;  // qp.hpp:193
    while (Grp<L>::warp_any(!done)) {
        if (!done && iter >= max_iterations) {
            status = kQpIterLimit;
            done = true;
        }
        // Most violated inactive row (qp.hpp:225-239).
        Real worst = tol;
        int p = -1;
        rows.scan(g, ux, uy, worst, p);
        g.argmax(worst, p);
        if (!done && p < 0) done = true;
        if (!Grp<L>::warp_any(!done)) break;  // every env of the warp is optimal
        bool act = !done;
        Real gx, gy, hp;
        rows.fetch(g, act ? p : rows.dummy_row(), gx, gy, hp);
        if (!vl) gx = Real(0);
        if (!vly) gy = Real(0);
        // Zero-norm violated row: b < 0 on a vacuous row (qp.hpp:242-253).
        const Real gn = g.sum(gx * gx + gy * gy);
        if (act && gn < Prec<Real>::eps_row) {
            status = kQpInfeasible;
            done = true;
            act = false;
        }
        if (act && vl) ws.gS[2 * lane] = gx;
        if (act && vly) ws.gS[2 * lane + 1] = gy;
        Grp<L>::sync();
        bool in = act, added = false;
        Real lam_p = 0;
        int guard = 0;
        if (__all_sync(Grp<L>::kFull, !act || k == 0)) {
            // Every active group enters its first row: the inner loop of
            // qp.hpp:262-330 with an empty active set, specialised (c = r = 0,
            // z = g, t1 = inf). Same arithmetic as the general path.
            const Real z2 = gn;  // same reduction as the general path's |z|^2 with z = g
            const Real viol = g.sum(gx * ux + gy * uy) - hp;
            if (act) {
                if (viol > tol && z2 > Prec<Real>::eps_z) {
                    const Real t = viol / z2;  // t = min(inf, t2)
                    ux -= t * gx;
                    uy -= t * gy;
                    const Real rho = dsqrt(z2);
                    const Real irho = Real(1) / rho;
                    if (vl) ws.Q[2 * lane] = gx * irho;
                    if (vly) ws.Q[2 * lane + 1] = gy * irho;
                    if (lane == 0) {
                        ws.R[0] = rho;
                        ws.Rd[0] = irho;
                        sl.lam0 = t;
                        sl.act0 = p;
                    }
                    rows.set_active(g, p, true);
                    k = 1;
                } else if (viol > tol) {  // dependent normal, nothing blocks: infeasible (qp.hpp:304-309)
                    status = kQpInfeasible;
                    done = true;
                }
                added = true;  // (viol <= tol: finished without adding, lam_p == 0)
            }
            Grp<L>::sync();
            in = false;
        }
        while (Grp<L>::warp_any(in)) {  // qp.hpp:262-330
            // c = Q^T g on this lane's slots
            sl.c0 = sl.c1 = Real(0);
            if (in) {
                if (a0 < k) {
                    Real c = 0;
                    for (int v = 0; v < n; ++v) c += ws.Q[a0 * n + v] * ws.gS[v];
                    sl.c0 = c;
                    ws.cS[a0] = c;
                }
                if (a1 < k) {  // (slots >= L only exist for N > L/2 ... k > L)
                    Real c = 0;
                    for (int v = 0; v < n; ++v) c += ws.Q[a1 * n + v] * ws.gS[v];
                    sl.c1 = c;
                    ws.cS[a1] = c;
                }
            }
            Grp<L>::sync();
            // z = g - Q c (this lane's two components)
            Real zx = gx, zy = gy;
            if (in && vl) {
                for (int a = 0; a < k; ++a) {
                    const Real ca = ws.cS[a];
                    zx -= ws.Q[a * n + 2 * lane] * ca;
                    if (vly) zy -= ws.Q[a * n + 2 * lane + 1] * ca;
                }
            }
            // r = R^{-1} c: column-oriented back substitution, r_b broadcast by shuffle
            sl.r0 = sl.c0;
            sl.r1 = sl.c1;
            const int kmax = Grp<L>::warp_max(in ? k : 0);
            for (int b = kmax - 1; b >= 0; --b) {
                const bool hi = b >= L;
                const Real rb = g.shfl(hi ? sl.r1 : sl.r0, b & (L - 1)) * ws.Rd[b];
                if (in && b < k) {
                    if (a0 == b) sl.r0 = rb;
                    else if (a0 < b) sl.r0 -= ws.R[b * n + a0] * rb;
                    if (a1 == b) sl.r1 = rb;
                    else if (a1 < b) sl.r1 -= ws.R[b * n + a1] * rb;
                }
            }
            const Real z2 = g.sum(zx * zx + zy * zy);
            const Real viol = g.sum(gx * ux + gy * uy) - hp;  // qp.hpp:281
            // First blocking multiplier (qp.hpp:291-302).
            Real t1 = Consts<Real>::inf;
            int bi = -1;
            if (in) {
                if (a0 < k && sl.r0 > Prec<Real>::eps_r) {
                    t1 = sl.lam0 / sl.r0;
                    bi = a0;
                }
                if (a1 < k && sl.r1 > Prec<Real>::eps_r) {
                    const Real t = sl.lam1 / sl.r1;
                    if (bi < 0 || t < t1) {
                        t1 = t;
                        bi = a1;
                    }
                }
            }
            g.argmin(t1, bi);
            if (bi < 0) t1 = Consts<Real>::inf;
            bool finish = false, do_add = false, do_drop = false, infeas = false, step_u = false, step_l = false;
            Real t = 0;
            if (in) {
                if (viol <= tol) {  // qp.hpp:282-289
                    finish = true;
                    do_add = lam_p > Real(0) && z2 > Prec<Real>::eps_z;
                } else if (z2 <= Prec<Real>::eps_z) {  // qp.hpp:304-315
                    if (bi < 0) {
                        infeas = true;
                    } else {
                        t = t1;
                        step_l = true;
                        do_drop = true;
                    }
                } else {  // qp.hpp:317-329
                    const Real t2 = viol / z2;
                    t = dmin(t1, t2);
                    step_u = step_l = true;
                    if (t2 <= t1) {
                        do_add = true;
                        finish = true;
                    } else {
                        do_drop = true;
                    }
                }
            }
            if (step_u) {
                ux -= t * zx;
                uy -= t * zy;
            }
            if (step_l) {
                if (a0 < k) sl.lam0 -= t * sl.r0;
                if (a1 < k) sl.lam1 -= t * sl.r1;
                lam_p += t;
            }
            if (do_add) {
                const Real rho = dsqrt(z2);
                const Real irho = Real(1) / rho;
                if (vl) ws.Q[k * n + 2 * lane] = zx * irho;
                if (vly) ws.Q[k * n + 2 * lane + 1] = zy * irho;
                if (a0 < k) ws.R[k * n + a0] = sl.c0;
                if (a1 < k) ws.R[k * n + a1] = sl.c1;
                if (lane == 0) {
                    ws.R[k * n + k] = rho;
                    ws.Rd[k] = irho;
                }
                if (a0 == k) {
                    sl.lam0 = lam_p;
                    sl.act0 = p;
                }
                if (a1 == k) {
                    sl.lam1 = lam_p;
                    sl.act1 = p;
                }
                rows.set_active(g, p, true);
                ++k;
            }
            qp_drop<Real, L>(g, rows, ws, sl, n, k, do_drop, bi);
            if (finish) {
                in = false;
                added = true;
            }
            if (infeas) {
                in = false;
                status = kQpInfeasible;
                done = true;
            }
            ++guard;
            if (in && guard > total_rows) in = false;  // guard exhausted without adding
            Grp<L>::sync();
        }
        if (act && !added) done = true;  // stall (qp.hpp:331-334) or infeasible
        if (act) ++iter;
    }
    return status;
}

// ---------------------------------------------------------------------------
// Dense rows (unit-level entry point, fold_rows qp.hpp:104-141): row r of A
// in smem, normalised; finite box sides folded after the rows in variable
// order, hi before lo. Row r is scanned by lane r % L; active sets are
// group-uniform bit masks.
// ---------------------------------------------------------------------------
template <class Real, int L, int MAXM>
struct DenseRows {
    const Real* G;    // [m][n] normalised rows (smem)
    const Real* h;    // [m]
    Real* ush;        // [n] u broadcast scratch (smem)
    const Real* lo;   // [n] box (+-1e30 = unbounded)
    const Real* hi;
    int n, m;
    unsigned long long active_rows;  // bit r: row r active (group-uniform)
    unsigned long long box_active;   // bit 2v (hi) / 2v+1 (lo)

    __device__ int dummy_row() const { return 0; }

    __device__ void scan(const Grp<L>& g, Real ux, Real uy, Real& worst, int& p) {
        const int lane = g.lane;
        if (2 * lane < n) ush[2 * lane] = ux;
        if (2 * lane + 1 < n) ush[2 * lane + 1] = uy;
        Grp<L>::sync();
        for (int r = lane; r < m; r += L) {
            if ((active_rows >> r) & 1ull) continue;
            Real s = 0;
            for (int i = 0; i < n; ++i) s += G[r * n + i] * ush[i];
            const Real v = s - h[r];
            if (v > worst) {
                worst = v;
                p = r;
            }
        }
        if (2 * lane < n) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int v = 2 * lane + c;
                if (v >= n) continue;
                const Real u = c ? uy : ux;
                if (hi[v] < Real(1e30) && !((box_active >> (2 * v)) & 1ull)) {
                    const Real val = u - hi[v];
                    if (val > worst) { worst = val; p = m + 2 * v; }
                }
                if (lo[v] > Real(-1e30) && !((box_active >> (2 * v + 1)) & 1ull)) {
                    const Real val = -u + lo[v];
                    if (val > worst) { worst = val; p = m + 2 * v + 1; }
                }
            }
        }
        Grp<L>::sync();
    }
    __device__ void fetch(const Grp<L>& g, int p, Real& gx, Real& gy, Real& hp) const {
        const int lane = g.lane;
        gx = gy = Real(0);
        if (p < m) {
            if (2 * lane < n) gx = G[p * n + 2 * lane];
            if (2 * lane + 1 < n) gy = G[p * n + 2 * lane + 1];
            hp = h[p];
        } else {
            const int q = p - m;
            const int v = q >> 1;
            const bool is_lo = q & 1;
            const Real s = is_lo ? Real(-1) : Real(1);
            if (lane == (v >> 1)) {
                if (v & 1) gy = s;
                else gx = s;
            }
            hp = is_lo ? -lo[v] : hi[v];
        }
    }
    __device__ void set_active(const Grp<L>&, int p, bool on) {
        if (p < m) {
            if (on) active_rows |= 1ull << p;
            else active_rows &= ~(1ull << p);
        } else {
            const int q = p - m;
            if (on) box_active |= 1ull << q;
            else box_active &= ~(1ull << q);
        }
    }
};

}  // namespace mrsim_dev
