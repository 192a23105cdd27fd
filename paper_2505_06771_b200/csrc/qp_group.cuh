// qp_group.cuh — the CBF safety QP, solved cooperatively by the L lanes of
// one environment group.
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
//   * lane v owns variable v (u_v, g_v, z_v); lane a owns active slot a
//     (c_a, r_a, lambda_a). Reductions are butterfly shuffles in the group.
//   * rows are never materialised in HBM: the RowSet policy evaluates them
//     on the fly (barrier rows from the robots' projected points, or dense
//     rows for the unit-level entry point).
#pragma once

#include "mrsim_device.cuh"

namespace mrsim_dev {

enum QpStatusDev : int { kQpOptimal = 0, kQpInfeasible = 1, kQpIterLimit = 2 };

// Shared-memory workspace of one group for n <= L variables.
//   Q: column a (active slot a) at Q + a*(n+1), indexed by variable
//   R: R[row][col] at R + col*(n+1) + row (upper triangular)
//   gp, c: broadcast scratch [n]; act: active row indices [n]
template <class Real>
struct QpSmem {
    Real* Q;
    Real* R;
    Real* gp;
    Real* c;
    int* act;
    static __host__ __device__ constexpr int reals(int n) { return 2 * n * (n + 1) + 2 * n; }
    static __host__ __device__ constexpr int ints(int n) { return n; }
    __device__ void carve(Real* base, int* ibase, int n) {
        Q = base;
        R = Q + n * (n + 1);
        gp = R + n * (n + 1);
        c = gp + n;
        act = ibase;
    }
};

// Drop active slot b: delete column b of N = Q R and restore triangularity
// with Givens rotations (the reference erases active[b] / lambda[b] and
// re-factorises, qp.hpp:270-271, 312-313, 327-328; order is preserved).
template <class Real, int L, class RowSet>
__device__ __forceinline__ void qp_drop(const Group<L>& g, RowSet& rows, const QpSmem<Real>& ws, int n, int& k,
                                        Real& lam, int b) {
    const int lane = g.lane;
    const int s = n + 1;
    rows.set_active(g, ws.act[b], false);
    // shift multipliers and active indices down over slot b
    const Real lam_up = g.shfl(lam, lane + 1 < L ? lane + 1 : lane);
    int act_up = (lane + 1 < k) ? ws.act[lane + 1] : 0;
    g.sync();
    if (lane >= b && lane < k - 1) {
        lam = lam_up;
        ws.act[lane] = act_up;
    }
    // delete column b of R (lane = row)
    if (lane < k) {
        for (int col = b; col < k - 1; ++col) ws.R[col * s + lane] = ws.R[(col + 1) * s + lane];
    }
    g.sync();
    for (int j = b; j < k - 1; ++j) {
        const Real a = ws.R[j * s + j];
        const Real bb = ws.R[j * s + j + 1];
        g.sync();
        const Real rho = dhypot(a, bb);
        const Real cg = a / rho, sg = bb / rho;
        if (lane >= j && lane < k - 1) {  // rows j, j+1 of R, column = lane
            const Real x = ws.R[lane * s + j], y = ws.R[lane * s + j + 1];
            ws.R[lane * s + j] = cg * x + sg * y;
            ws.R[lane * s + j + 1] = (lane == j) ? Real(0) : (-sg * x + cg * y);
        }
        if (lane < n) {  // columns j, j+1 of Q, row = lane
            const Real x = ws.Q[j * s + lane], y = ws.Q[(j + 1) * s + lane];
            ws.Q[j * s + lane] = cg * x + sg * y;
            ws.Q[(j + 1) * s + lane] = -sg * x + cg * y;
        }
        g.sync();
    }
    --k;
}

// Solve. `u` holds u_v on lane v < n (in: u_nom, out: solution).
template <class Real, int L, class RowSet>
__device__ int qp_solve_group(const Group<L>& g, RowSet& rows, const QpSmem<Real>& ws, int n, Real& u,
                              int total_rows, int max_iterations, Real tol, int* iterations_out) {
    const int lane = g.lane;
    const int s = n + 1;
    int k = 0;     // active-set size (uniform across the group)
    Real lam = 0;  // lane a < k: lambda_a
    if (max_iterations <= 0) max_iterations = 100 + 20 * total_rows;  // qp.hpp:193
    int iter = 0;
    int status = kQpOptimal;
    for (; iter < max_iterations; ++iter) {
        // Most violated inactive row (qp.hpp:225-239).
        Real worst = tol;
        int p = -1;
        rows.scan(g, u, worst, p);
        g.argmax(worst, p);
        if (p < 0) break;

        Real gp, hp;  // lane v: component v of row p; rhs (uniform)
        rows.fetch(g, p, gp, hp);
        if (lane >= n) gp = 0;
        // Zero-norm violated row: b < 0 on a vacuous row (qp.hpp:242-253).
        if (g.sum(gp * gp) < Prec<Real>::eps_row) {
            status = kQpInfeasible;
            break;
        }
        if (lane < n) ws.gp[lane] = gp;
        g.sync();

        bool added = false;
        Real lam_p = 0;
        for (int guard = 0; guard <= total_rows && !added; ++guard) {  // qp.hpp:262
            // c = Q^T g_p on lane a < k
            Real ca = 0;
            if (lane < k) {
                const Real* qa = ws.Q + lane * s;
                for (int v = 0; v < n; ++v) ca += qa[v] * ws.gp[v];
                ws.c[lane] = ca;
            }
            g.sync();
            // z = g_p - Q c on lane v < n
            Real z = 0;
            if (lane < n) {
                z = gp;
                for (int a = 0; a < k; ++a) z -= ws.Q[a * s + lane] * ws.c[a];
            }
            // r = R^{-1} c (back substitution, column oriented)
            Real ra = ca;
            for (int b = k - 1; b >= 0; --b) {
                if (lane == b) ra = ra / ws.R[b * s + b];
                const Real rb = g.shfl(ra, b);
                if (lane < b) ra -= ws.R[b * s + lane] * rb;
            }
            const Real z2 = g.sum(z * z);
            const Real viol = g.sum(lane < n ? gp * u : Real(0)) - hp;  // qp.hpp:281
            if (viol <= tol) {  // qp.hpp:282-289
                if (lam_p > Real(0) && z2 > Prec<Real>::eps_z) {
                    const Real rho = dsqrt(z2);
                    if (lane < n) ws.Q[k * s + lane] = z / rho;
                    if (lane < k) ws.R[k * s + lane] = ca;
                    if (lane == k) {
                        ws.R[k * s + k] = rho;
                        lam = lam_p;
                        ws.act[k] = p;
                    }
                    rows.set_active(g, p, true);
                    ++k;
                }
                g.sync();
                added = true;
                break;
            }
            // First blocking multiplier (qp.hpp:291-302).
            Real t1 = Consts<Real>::inf;
            int blocker = -1;
            if (lane < k && ra > Prec<Real>::eps_r) {
                t1 = lam / ra;
                blocker = lane;
            }
            g.argmin(t1, blocker);
            if (blocker < 0) t1 = Consts<Real>::inf;
            if (z2 <= Prec<Real>::eps_z) {  // qp.hpp:304-315
                if (blocker < 0) {
                    status = kQpInfeasible;
                    if (iterations_out) *iterations_out = iter;
                    return status;
                }
                if (lane < k) lam -= t1 * ra;
                lam_p += t1;
                qp_drop<Real, L>(g, rows, ws, n, k, lam, blocker);
                continue;
            }
            const Real t2 = viol / z2;  // qp.hpp:317-329
            const Real t = dmin(t1, t2);
            if (lane < n) u -= t * z;
            if (lane < k) lam -= t * ra;
            lam_p += t;
            if (t2 <= t1) {
                const Real rho = dsqrt(z2);
                if (lane < n) ws.Q[k * s + lane] = z / rho;
                if (lane < k) ws.R[k * s + lane] = ca;
                if (lane == k) {
                    ws.R[k * s + k] = rho;
                    lam = lam_p;
                    ws.act[k] = p;
                }
                rows.set_active(g, p, true);
                ++k;
                g.sync();
                added = true;
            } else {
                qp_drop<Real, L>(g, rows, ws, n, k, lam, blocker);
            }
        }
        if (!added) break;  // stall (qp.hpp:331-334)
    }
    if (status == kQpOptimal && iter >= max_iterations) status = kQpIterLimit;
    if (iterations_out) *iterations_out = iter;
    return status;
}

// ---------------------------------------------------------------------------
// Dense rows (unit-level entry point, fold_rows qp.hpp:104-141): row r of A
// in smem, normalised; finite box sides folded after the rows in variable
// order, hi before lo. Owner of row r: lane r % L.
// ---------------------------------------------------------------------------
template <class Real, int L, int MAXM>
struct DenseRows {
    static constexpr int kSlots = (MAXM + L - 1) / L;
    const Real* G;  // [m][n] normalised rows (smem)
    const Real* h;  // [m]
    Real* ush;      // [n] u broadcast scratch (smem)
    const Real* lo;  // [n] box (global, +-1e30 = unbounded)
    const Real* hi;
    int n, m;
    unsigned long long active_rows;  // bit r: row r active (uniform)
    unsigned box_active;             // bit 2v (hi) / 2v+1 (lo) (uniform)

    __device__ void scan(const Group<L>& g, Real u, Real& worst, int& p) {
        if (g.lane < n) ush[g.lane] = u;
        g.sync();
        for (int sl = 0; sl < kSlots; ++sl) {
            const int r = g.lane + sl * L;
            if (r < m && !((active_rows >> r) & 1ull)) {
                Real s = 0;
                for (int i = 0; i < n; ++i) s += G[r * n + i] * ush[i];
                const Real v = s - h[r];
                if (v > worst) { worst = v; p = r; }
            }
        }
        if (g.lane < n) {
            const int v = g.lane;
            if (hi[v] < Real(1e30) && !((box_active >> (2 * v)) & 1u)) {
                const Real val = u - hi[v];
                if (val > worst) { worst = val; p = m + 2 * v; }
            }
            if (lo[v] > Real(-1e30) && !((box_active >> (2 * v + 1)) & 1u)) {
                const Real val = -u + lo[v];
                if (val > worst) { worst = val; p = m + 2 * v + 1; }
            }
        }
        g.sync();
    }
    __device__ void fetch(const Group<L>& g, int p, Real& gv, Real& hp) const {
        if (p < m) {
            gv = g.lane < n ? G[p * n + g.lane] : Real(0);
            hp = h[p];
        } else {
            const int q = p - m;
            const int v = q >> 1;
            const bool is_lo = q & 1;
            gv = (g.lane == v) ? (is_lo ? Real(-1) : Real(1)) : Real(0);
            hp = is_lo ? -lo[v] : hi[v];
        }
    }
    __device__ void set_active(const Group<L>&, int p, bool on) {
        if (p < m) {
            if (on) active_rows |= 1ull << p;
            else active_rows &= ~(1ull << p);
        } else {
            const int q = p - m;
            if (on) box_active |= 1u << q;
            else box_active &= ~(1u << q);
        }
    }
};

}  // namespace mrsim_dev
