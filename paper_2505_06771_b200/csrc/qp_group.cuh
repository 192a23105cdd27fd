// qp_group.cuh — the CBF safety QP, solved cooperatively by the L lanes of
// one environment group, in warp lockstep (see group.cuh).
//
//   minimize 0.5 ||u - u_nom||^2   s.t.  g_r . u <= h_r   (unit-norm rows)
//
// Same algorithm and the same discrete decisions as the reference's
// solve_qp (qp.hpp:183-357): Goldfarb-Idnani dual active set with H = I,
// most-violated row first (ties -> lowest row index), partial dual steps
// that drop the first blocking multiplier, infeasibility when the entering
// normal is dependent and nothing blocks. The reference re-forms the Gram
// matrix M = N^T N of the active normals and Cholesky-solves it at every
// inner step (qp.hpp:199-221). Here the inverse Gram matrix S = M^{-1} is
// kept up to date instead:
//   r   = S (N^T g)                        (one parallel mat-vec, no sequential solve)
//   z   = g - N r                          (|z|^2 is the Schur complement of M + g)
//   add : S <- [[S + r r^T / s, -r / s], [-r^T / s, 1 / s]],  s = |z|^2
//   drop: S <- S_{-b,-b} - S_{-b,b} S_{b,-b} / S_bb           (rank-1 downdate)
// Rows are used through small descriptors (a barrier row touches at most two
// robots), so N^T g and N r cost O(k) per lane. Slots are addressed through a
// logical->physical permutation so a drop never moves S; the logical order
// (= the reference's active-list order) drives the tie-breaks.
//
// Lane l owns variables 2l, 2l+1 (one robot) and logical slots l, l+L.
// Every loop that contains a collective has a warp-uniform trip count and
// per-environment decisions are predicates, so the warp (32/L environments)
// runs in lockstep with full-mask shuffles.
#pragma once

#include "group.cuh"
#include "mrsim_device.cuh"

namespace mrsim_dev {

enum QpStatusDev : int { kQpOptimal = 0, kQpInfeasible = 1, kQpIterLimit = 2 };


// Shared-memory workspace of one group for n variables (all indexed by
// PHYSICAL slot unless noted):
//   S[q*n + q'] inverse Gram, lam, r, d, act (row id), desc (row descriptor),
//   pm[a] logical -> physical (a permutation; entries >= k are free slots)
template <class Real, class Desc>
struct QpWs {
    Real *S, *lam, *r, *d;
    int *act, *pm;
    Desc* desc;
    static __host__ __device__ constexpr int bytes(int n) {
        return static_cast<int>(sizeof(Real)) * (n * n + 3 * n) + 8 * n + static_cast<int>(sizeof(Desc)) * n;
    }
    __device__ void carve(unsigned char* base, int n) {
        S = reinterpret_cast<Real*>(base);
        lam = S + n * n;
        r = lam + n;
        d = r + n;
        desc = reinterpret_cast<Desc*>(d + n);
        act = reinterpret_cast<int*>(desc + n);
        pm = act + n;
    }
};

// Solve for the groups with `participate` set. (ux, uy): this lane's pair of
// variables (in: u_nom, out: solution). Returns the QpStatusDev of the group.
// FAST: specialise the first entering row when the whole warp starts from an
// empty active set (same arithmetic; a speed/register-pressure trade chosen
// per task, see qp_fast_first_row in step_kernel.cuh).
template <class Real, int L, bool FAST = true, class RowSet>
__device__ __forceinline__ int qp_solve(const Grp<L>& g, RowSet& rows, const QpWs<Real, typename RowSet::Desc>& ws,
                                        int n, bool participate, Real& ux, Real& uy, int total_rows, Real tol) {
    typedef typename RowSet::Desc Desc;
    const int lane = g.lane;
    const bool vl = 2 * lane < n;      // this lane's x variable exists
    const bool vly = 2 * lane + 1 < n;  // ... and its y variable (n may be odd for dense QPs)
    const int a0 = lane, a1 = lane + L;  // this lane's logical slots
    for (int a = lane; a < n; a += L) ws.pm[a] = a;
    int k = 0;
    unsigned tm = 0;  // physical slots whose row touches this lane's variables (n <= 32)
    int status = kQpOptimal;
    bool done = !participate;
    int iter = 0;
    const int max_iterations = 100 + 20 * total_rows;  // qp.hpp:193
    Grp<L>::sync();
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
        const Desc gd = rows.describe(g, act ? p : rows.dummy_row());
        Real gx, gy;
        rows.comp(gd, lane, gx, gy);
        const Real hp = rows.rhs(gd);
        if (!vl) gx = Real(0);
        if (!vly) gy = Real(0);
        // Zero-norm violated row: b < 0 on a vacuous row (qp.hpp:242-253).
        const Real gn = g.sum(gx * gx + gy * gy);
        if (act && gn < Prec<Real>::eps_row) {
            status = kQpInfeasible;
            done = true;
            act = false;
        }
        bool in = act, added = false;
        Real lam_p = 0;
        int guard = 0;
        if (FAST && __all_sync(Grp<L>::kFull, !act || k == 0)) {
            // Every active group enters its first row: the inner loop below with
            // an empty active set (r = 0, z = g, |z|^2 = gn, t1 = inf), same arithmetic.
            const Real viol = g.sum(gx * ux + gy * uy) - hp;
            if (act) {
                if (viol <= tol) {
                    added = true;  // finish, nothing to add (lam_p = 0)
                } else if (gn <= Prec<Real>::eps_z) {
                    status = kQpInfeasible;  // dependent normal, nothing blocks (qp.hpp:304-309)
                    done = true;
                } else {
                    const Real t = viol / gn;
                    ux -= t * gx;
                    uy -= t * gy;
                    const int qk = ws.pm[0];
                    if (rows.touches(gd, lane)) tm |= 1u << qk;
                    if (lane == 0) {
                        ws.S[qk * n + qk] = Real(1) / gn;
                        ws.lam[qk] = t;
                        ws.act[qk] = p;
                        ws.desc[qk] = gd;
                    }
                    rows.set_active(g, p, true);
                    k = 1;
                    added = true;
                }
            }
            in = false;
            Grp<L>::sync();
        }
        while (Grp<L>::warp_any(in)) {  // qp.hpp:262-330
            // d = N^T g on this lane's logical slots (physical q)
            const int q0 = (in && a0 < k) ? ws.pm[a0] : 0;
            const int q1 = (in && a1 < k) ? ws.pm[a1] : 0;
            if (in && a0 < k) ws.d[q0] = rows.dot(ws.desc[q0], gd);
            if (in && a1 < k) ws.d[q1] = rows.dot(ws.desc[q1], gd);
            Grp<L>::sync();
            // r = S d (qp.hpp:264's solve_gram, as a mat-vec)
            Real r0 = 0, r1 = 0;
            if (in && a0 < k) {
                for (int c = 0; c < k; ++c) {
                    const int qc = ws.pm[c];
                    r0 += ws.S[q0 * n + qc] * ws.d[qc];
                }
                ws.r[q0] = r0;
            }
            if (in && a1 < k) {
                for (int c = 0; c < k; ++c) {
                    const int qc = ws.pm[c];
                    r1 += ws.S[q1 * n + qc] * ws.d[qc];
                }
                ws.r[q1] = r1;
            }
            Grp<L>::sync();
            // z = g - N r (this lane's two components)
            Real zx = gx, zy = gy;
            if (in && vl) {
                for (unsigned m = tm; m; m &= m - 1) {  // only the active rows touching this lane's variables
                    const int qc = __ffs(m) - 1;
                    Real cx, cy;
                    rows.comp(ws.desc[qc], lane, cx, cy);
                    const Real rc = ws.r[qc];
                    zx -= rc * cx;
                    zy -= rc * cy;
                }
            }
            if (!vly) zy = Real(0);
            const Real z2 = g.sum(zx * zx + zy * zy);
            const Real viol = g.sum(gx * ux + gy * uy) - hp;  // qp.hpp:281
            // First blocking multiplier in logical order (qp.hpp:291-302).
            Real t1 = Consts<Real>::inf;
            int bi = -1;
            if (in) {
                if (a0 < k && r0 > Prec<Real>::eps_r) {
                    t1 = ws.lam[q0] / r0;
                    bi = a0;
                }
                if (a1 < k && r1 > Prec<Real>::eps_r) {
                    const Real t = ws.lam[q1] / r1;
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
                if (a0 < k) ws.lam[q0] -= t * r0;
                if (a1 < k) ws.lam[q1] -= t * r1;
                lam_p += t;
            }
            if (do_add) {  // bordered inverse: the new slot's Schur complement is |z|^2
                const Real is = Real(1) / z2;
                const int qk = ws.pm[k];
                for (int a = lane; a < k; a += L) {
                    const int qa = ws.pm[a];
                    const Real ra = ws.r[qa];
                    for (int c = 0; c < k; ++c) {
                        const int qc = ws.pm[c];
                        ws.S[qa * n + qc] += ra * ws.r[qc] * is;
                    }
                    ws.S[qa * n + qk] = -ra * is;
                    ws.S[qk * n + qa] = -ra * is;
                }
                if (rows.touches(gd, lane)) tm |= 1u << qk;
                if (lane == 0) {
                    ws.S[qk * n + qk] = is;
                    ws.lam[qk] = lam_p;
                    ws.act[qk] = p;
                    ws.desc[qk] = gd;
                }
                rows.set_active(g, p, true);
                ++k;
            }
            Grp<L>::sync();
            if (do_drop) {  // S <- S_{-b,-b} - S_{-b,b} S_{b,-b} / S_bb, then free the slot
                const int qb = ws.pm[bi];
                tm &= ~(1u << qb);
                rows.set_active(g, ws.act[qb], false);
                const Real ib = Real(1) / ws.S[qb * n + qb];
                for (int a = lane; a < k; a += L) {
                    if (a == bi) continue;
                    const int qa = ws.pm[a];
                    const Real sab = ws.S[qa * n + qb] * ib;
                    for (int c = 0; c < k; ++c) {
                        if (c == bi) continue;
                        const int qc = ws.pm[c];
                        ws.S[qa * n + qc] -= sab * ws.S[qb * n + qc];
                    }
                }
            }
            // logical order: slots after bi move down by one, the freed slot goes to the end
            int pm_next0 = 0, pm_next1 = 0;
            const bool m0 = do_drop && a0 >= bi && a0 < k - 1;
            const bool m1 = do_drop && a1 >= bi && a1 < k - 1;
            if (m0) pm_next0 = ws.pm[a0 + 1];
            if (m1) pm_next1 = ws.pm[a1 + 1];
            const int freed = do_drop ? ws.pm[bi] : 0;
            Grp<L>::sync();
            if (m0) ws.pm[a0] = pm_next0;
            if (m1) ws.pm[a1] = pm_next1;
            if (do_drop && lane == ((k - 1) & (L - 1))) ws.pm[k - 1] = freed;
            if (do_drop) --k;
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
// group-uniform bit masks. A descriptor is the row index.
// ---------------------------------------------------------------------------
template <class Real, int L, int MAXM>
struct DenseRows {
    struct Desc {
        int p;
    };
    const Real* G;    // [m][n] normalised rows (smem)
    const Real* h;    // [m]
    Real* ush;        // [n] u broadcast scratch (smem)
    const Real* lo;   // [n] box (+-1e30 = unbounded)
    const Real* hi;
    int n, m;
    unsigned long long active_rows;  // bit r: row r active (group-uniform)
    unsigned long long box_active;   // bit 2v (hi) / 2v+1 (lo)

    __device__ int dummy_row() const { return 0; }
    __device__ Desc describe(const Grp<L>&, int p) const { return Desc{p}; }
    // component of row p on variable v
    __device__ Real at(int p, int v) const {
        if (v >= n) return Real(0);
        if (p < m) return G[p * n + v];
        const int q = p - m;
        return (v == (q >> 1)) ? ((q & 1) ? Real(-1) : Real(1)) : Real(0);
    }
    __device__ void comp(const Desc& dsc, int lane, Real& cx, Real& cy) const {
        cx = at(dsc.p, 2 * lane);
        cy = at(dsc.p, 2 * lane + 1);
    }
    __device__ static bool touches(const Desc&, int) { return true; }
    __device__ Real rhs(const Desc& dsc) const {
        if (dsc.p < m) return h[dsc.p];
        const int q = dsc.p - m, v = q >> 1;
        return (q & 1) ? -lo[v] : hi[v];
    }
    __device__ Real dot(const Desc& a, const Desc& b) const {
        Real s = 0;
        for (int v = 0; v < n; ++v) s += at(a.p, v) * at(b.p, v);
        return s;
    }

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
