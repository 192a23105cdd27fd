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

// Diagnostic counters (builds with -DMRSIM_QP_STATS only): [0] solves, [1] warm attempts,
// [2] warm fallbacks (dependent), [3] warm fallbacks (negative multiplier), [4] outer iterations.
#ifdef MRSIM_QP_STATS
__device__ unsigned long long g_qp_stats[8];
#define MRSIM_QP_STAT(i, cond) \
    do {                          \
        if (cond) atomicAdd(&g_qp_stats[i], 1ull); \
    } while (0)
#else
#define MRSIM_QP_STAT(i, cond) \
    do {                          \
    } while (0)
#endif


// Shared-memory workspace of one group for n variables, indexed by PHYSICAL
// slot: S[q*n + q'] inverse Gram, lam, r, d, act (row id), desc (row descriptor).
// Physical slot q is owned by lane q % L (q < 2L); the owner keeps the slot's
// logical position (= the reference's active-list order,
// which drives the tie-breaks) in registers, so a drop never moves data.
template <class Real, class Desc>
struct QpWs {
    Real *S, *lam, *r, *d;
    Desc* desc;
    int* act;
    int* warm;  // the group's previous active rows, in logical order (warm-started entering order)
    static constexpr int kGuardBytes = 4 * MRSIM_GUARD_WORDS;  // checks builds: a guard behind each array
    static __host__ __device__ constexpr int bytes(int n) {
        return static_cast<int>(sizeof(Real)) * (n * n + 3 * n) + static_cast<int>(sizeof(Desc)) * n + 8 * n +
               7 * kGuardBytes;
    }
    __device__ void carve(unsigned char* base, int n) {
        S = reinterpret_cast<Real*>(base);
#if MRSIM_GUARD_WORDS
        lam = reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(S + n * n) + kGuardBytes);
        r = reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(lam + n) + kGuardBytes);
        d = reinterpret_cast<Real*>(reinterpret_cast<unsigned char*>(r + n) + kGuardBytes);
        desc = reinterpret_cast<Desc*>(reinterpret_cast<unsigned char*>(d + n) + kGuardBytes);
        act = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(desc + n) + kGuardBytes);
        warm = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(act + n) + kGuardBytes);
#else
        lam = S + n * n;
        r = lam + n;
        d = r + n;
        desc = reinterpret_cast<Desc*>(d + n);
        act = reinterpret_cast<int*>(desc + n);
        warm = act + n;
#endif
    }
#if MRSIM_GUARD_WORDS
    // guard word g (0..7*4) of this workspace for n variables
    __device__ unsigned* guard(int n, int k) const {
        unsigned char* const ends[7] = {reinterpret_cast<unsigned char*>(S + n * n),
                                        reinterpret_cast<unsigned char*>(lam + n),
                                        reinterpret_cast<unsigned char*>(r + n),
                                        reinterpret_cast<unsigned char*>(d + n),
                                        reinterpret_cast<unsigned char*>(desc + n),
                                        reinterpret_cast<unsigned char*>(act + n),
                                        reinterpret_cast<unsigned char*>(warm + n)};
        return reinterpret_cast<unsigned*>(ends[k / MRSIM_GUARD_WORDS]) + k % MRSIM_GUARD_WORDS;
    }
#endif
};

// Checked slot index of the QP workspace (checks builds; no-op otherwise).
#define MRSIM_QP_SLOT_OK(q, n) MRSIM_DCHECK((q) >= 0 && (q) < (n))

// Solve for the groups with `participate` set. (ux, uy): this lane's pair of
// variables (in: u_nom, out: solution). Returns the QpStatusDev of the group.
// FAST: specialise the first entering row when the whole warp starts from an
// empty active set (same arithmetic; a speed/register-pressure trade chosen
// per task, see qp_fast_first_row in step_kernel.cuh).
//
// Warm start (WARM, warm_k != nullptr; Goldfarb-Idnani from a dual-feasible
// point): the rows active at the end of the group's previous solve (ws.warm,
// *warm_k of them, in their logical order) are re-entered on this tick's
// geometry by bordered-inverse updates alone (no scans, no steps), the
// multipliers of that set are solved directly, lam = S (N^T u_nom - h), and
// u = u_nom - N lam. If every multiplier is >= 0 this is a valid state of the
// dual method (dual feasible, the active rows tight), and the ordinary
// iteration continues from it: it adds whatever rows are still violated
// (usually none) and stops at the same unique optimum of the strictly convex
// QP as the cold start. A negative multiplier (the set changed) or a
// dependent row falls back to the cold start from u_nom.
template <class Real, int L, bool FAST = true, bool WARM = false, class RowSet>
__device__ __forceinline__ int qp_solve(const Grp<L>& g, RowSet& rows, const QpWs<Real, typename RowSet::Desc>& ws,
                                        int n, bool participate, Real& ux, Real& uy, int total_rows, Real tol,
                                        int* warm_k = nullptr) {
    typedef typename RowSet::Desc Desc;
    const int lane = g.lane;
    const bool vl = 2 * lane < n;      // this lane's x variable exists
    const bool vly = 2 * lane + 1 < n;  // ... and its y variable (n may be odd for dense QPs)
    const int q0 = lane, q1 = lane + L;  // this lane's physical slots (n <= 2L)
    int lp0 = -1, lp1 = -1;              // their logical positions, -1 = free
    unsigned amask = 0;                  // active physical slots (group-uniform; n <= 32)
    unsigned tm = 0;                     // active slots whose row touches this lane's variables
    int k = 0;
    int status = kQpOptimal;
    bool done = !participate;
    int iter = 0;
    const int max_iterations = 100 + 20 * total_rows;  // qp.hpp:193
    if constexpr (WARM) {
        const int wk = participate ? *warm_k : 0;  // previous active rows (group-uniform)
        MRSIM_DCHECK(wk >= 0 && wk <= n);
        const int wmax = Grp<L>::warp_max(wk);
        if (wmax > 0) {
            const Real ux0 = ux, uy0 = uy;
            bool wok = wk > 0;
            // 1) the previous active set on this tick's geometry: warm row j goes to physical slot j
            //    (= its logical position), owned by lane j % L
            for (int j = 0; j < wmax; ++j) {
                const bool act = wok && j < wk;
                const int pj = act ? ws.warm[j] : rows.dummy_row();
                const Desc gd = rows.describe(g, pj);
                if (act) {
                    if (lane == j % L) {
                        ws.act[j] = pj;
                        ws.desc[j] = gd;
                        if (j < L) lp0 = j;
                        else lp1 = j;
                    }
                    if (rows.touches(gd, lane)) tm |= 1u << j;
                    rows.set_active(g, pj, true);
                }
            }
            if (wok) {
                k = wk;
                amask = (k >= 32) ? ~0u : ((1u << k) - 1u);
            }
            Grp<L>::sync();
            //    M = N^T N of the set (each owner its rows), then S = M^-1 in place by Gauss-Jordan in
            //    logical order: M is SPD and the j-th pivot is the Schur complement |z|^2 the bordered
            //    update of row j would see, so `pivot <= eps_z` is the cold path's dependence test
            const bool w0 = wok && lp0 >= 0, w1 = wok && lp1 >= 0;
            // the warm set occupies physical slots [0, kw): counted loops (no mask walks)
            const int kw = wok ? wk : 0;
            if (w0)
                for (int c = 0; c < kw; ++c) ws.S[q0 * n + c] = rows.dot(ws.desc[q0], ws.desc[c]);
            if (w1)
                for (int c = 0; c < kw; ++c) ws.S[q1 * n + c] = rows.dot(ws.desc[q1], ws.desc[c]);
            for (int pv = 0; pv < wmax; ++pv) {
                Grp<L>::sync();
                const bool act = wok && pv < wk;
                const Real piv = act ? ws.S[pv * n + pv] : Real(1);
                if (act && !(piv > Prec<Real>::eps_z)) wok = false;  // dependent now: cold start
                const bool go = act && wok;
                Real* const prow = ws.S + pv * n;
                if (go && lane == pv % L) {  // scale the pivot row
                    const Real ip = Real(1) / piv;
#pragma unroll 4
                    for (int c = 0; c < kw; ++c) prow[c] *= ip;
                    prow[pv] = ip;
                }
                Grp<L>::sync();
                if (go) {  // eliminate the pivot column from the other rows
                    const Real ipv = prow[pv];
                    if (w0 && q0 != pv) {
                        Real* const row = ws.S + q0 * n;
                        const Real f = row[pv];
#pragma unroll 4
                        for (int c = 0; c < kw; ++c) row[c] = row[c] - f * prow[c];
                        row[pv] = -f * ipv;
                    }
                    if (w1 && q1 != pv) {
                        Real* const row = ws.S + q1 * n;
                        const Real f = row[pv];
#pragma unroll 4
                        for (int c = 0; c < kw; ++c) row[c] = row[c] - f * prow[c];
                        row[pv] = -f * ipv;
                    }
                }
            }
            Grp<L>::sync();
            // 2) lam = S (N^T u_nom - h), u = u_nom - N lam
            rows.publish_u(lane, ux0, uy0);
            Grp<L>::sync();
            if (w0) ws.d[q0] = rows.dot_u(ws.desc[q0]) - rows.rhs(ws.desc[q0]);
            if (w1) ws.d[q1] = rows.dot_u(ws.desc[q1]) - rows.rhs(ws.desc[q1]);
            Grp<L>::sync();
            Real l0 = 0, l1 = 0;
            if (w0 && wok) {
                for (int c = 0; c < kw; ++c) l0 += ws.S[q0 * n + c] * ws.d[c];
                ws.lam[q0] = l0;
            }
            if (w1 && wok) {
                for (int c = 0; c < kw; ++c) l1 += ws.S[q1 * n + c] * ws.d[c];
                ws.lam[q1] = l1;
            }
            // 3) dual feasibility of the warm point, else the cold start
            MRSIM_QP_STAT(1, lane == 0 && wk > 0);
            MRSIM_QP_STAT(2, lane == 0 && wk > 0 && !wok);
            if (g.any((w0 && wok && l0 < Real(0)) || (w1 && wok && l1 < Real(0)))) {
                MRSIM_QP_STAT(3, lane == 0 && wok);
                wok = false;
            }
            Grp<L>::sync();
            if (wok) {
                for (unsigned m = tm; m; m &= m - 1) {
                    const int c = __ffs(m) - 1;
                    Real cx, cy;
                    rows.comp(ws.desc[c], lane, cx, cy);
                    ux -= ws.lam[c] * cx;
                    uy -= ws.lam[c] * cy;
                }
                if (!vl) ux = Real(0);
                if (!vly) uy = Real(0);
            } else {  // cold start: empty active set at u_nom
                ux = ux0;
                uy = uy0;
                lp0 = lp1 = -1;
                amask = tm = 0u;
                k = 0;
                rows.active = 0u;
            }
            Grp<L>::sync();
        }
    }
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
        const bool touch = rows.touches(gd, lane);
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
                    if (lane == 0) {  // physical slot 0
                        ws.S[0] = Real(1) / gn;
                        ws.act[0] = p;
                        ws.desc[0] = gd;
                        ws.lam[0] = t;
                        lp0 = 0;
                    }
                    if (touch) tm = 1u;
                    amask = 1u;
                    rows.set_active(g, p, true);
                    k = 1;
                    added = true;
                }
            }
            in = false;
            Grp<L>::sync();
        }
        while (Grp<L>::warp_any(in)) {  // qp.hpp:262-330
            const bool s0 = in && lp0 >= 0, s1 = in && lp1 >= 0;  // own active slots
            MRSIM_DCHECK((!s0 || q0 < n) && (!s1 || q1 < n) && (n >= 32 || (amask >> n) == 0u));
            // d = N^T g
            if (s0) ws.d[q0] = rows.dot(ws.desc[q0], gd);
            if (s1) ws.d[q1] = rows.dot(ws.desc[q1], gd);
            Grp<L>::sync();
            // r = S d (qp.hpp:264's solve_gram, as a mat-vec)
            Real r0 = 0, r1 = 0;
            if (s0) {
                for (unsigned m = amask; m; m &= m - 1) {
                    const int c = __ffs(m) - 1;
                    r0 += ws.S[q0 * n + c] * ws.d[c];
                }
                ws.r[q0] = r0;
            }
            if (s1) {
                for (unsigned m = amask; m; m &= m - 1) {
                    const int c = __ffs(m) - 1;
                    r1 += ws.S[q1 * n + c] * ws.d[c];
                }
                ws.r[q1] = r1;
            }
            Grp<L>::sync();
            // z = g - N r (this lane's two components; only the rows touching them)
            Real zx = gx, zy = gy;
            if (in && vl) {
                for (unsigned m = tm; m; m &= m - 1) {
                    const int c = __ffs(m) - 1;
                    Real cx, cy;
                    rows.comp(ws.desc[c], lane, cx, cy);
                    const Real rc = ws.r[c];
                    zx -= rc * cx;
                    zy -= rc * cy;
                }
            }
            if (!vly) zy = Real(0);
            const Real z2 = g.sum(zx * zx + zy * zy);
            const Real viol = g.sum(gx * ux + gy * uy) - hp;  // qp.hpp:281
            // First blocking multiplier in logical order (qp.hpp:291-302):
            // key = logical position * 64 + physical slot.
            Real t1 = Consts<Real>::inf;
            int bk = -1;
            if (s0 && r0 > Prec<Real>::eps_r) {
                t1 = ws.lam[q0] / r0;
                bk = lp0 * 64 + q0;
            }
            if (s1 && r1 > Prec<Real>::eps_r) {
                const Real t = ws.lam[q1] / r1;
                const int key = lp1 * 64 + q1;
                if (bk < 0 || t < t1 || (t == t1 && key < bk)) {
                    t1 = t;
                    bk = key;
                }
            }
            g.argmin(t1, bk);
            const int bi = bk < 0 ? -1 : (bk >> 6);  // logical position of the blocking slot
            const int qb = bk < 0 ? 0 : (bk & 63);   // ... and its physical slot
            if (bk < 0) t1 = Consts<Real>::inf;
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
                if (s0) ws.lam[q0] -= t * r0;
                if (s1) ws.lam[q1] -= t * r1;
                lam_p += t;
            }
            if (do_add) {  // bordered inverse: the new slot's Schur complement is |z|^2
                const Real is = Real(1) / z2;
                const int qk = __ffs(~amask) - 1;  // lowest free physical slot
                MRSIM_QP_SLOT_OK(qk, n);
                if (s0) {
                    const Real ra = r0 * is;
                    for (unsigned m = amask; m; m &= m - 1) {
                        const int c = __ffs(m) - 1;
                        ws.S[q0 * n + c] += ra * ws.r[c];
                    }
                    ws.S[q0 * n + qk] = -ra;
                    ws.S[qk * n + q0] = -ra;
                }
                if (s1) {
                    const Real ra = r1 * is;
                    for (unsigned m = amask; m; m &= m - 1) {
                        const int c = __ffs(m) - 1;
                        ws.S[q1 * n + c] += ra * ws.r[c];
                    }
                    ws.S[q1 * n + qk] = -ra;
                    ws.S[qk * n + q1] = -ra;
                }
                if (lane == (qk & (L - 1))) {
                    ws.S[qk * n + qk] = is;
                    ws.act[qk] = p;
                    ws.desc[qk] = gd;
                    ws.lam[qk] = lam_p;
                    if (qk < L) lp0 = k;
                    else lp1 = k;
                }
                if (touch) tm |= 1u << qk;
                amask |= 1u << qk;
                rows.set_active(g, p, true);
                ++k;
            }
            if (do_drop) {  // S <- S_{-b,-b} - S_{-b,b} S_{b,-b} / S_bb; later slots move up one logical place
                MRSIM_DCHECK(qb < n && ((amask >> qb) & 1u));
                rows.set_active(g, ws.act[qb], false);
                const unsigned rest = amask & ~(1u << qb);
                const Real ib = Real(1) / ws.S[qb * n + qb];
                if (s0 && q0 != qb) {
                    const Real sab = ws.S[q0 * n + qb] * ib;
                    for (unsigned m = rest; m; m &= m - 1) {
                        const int c = __ffs(m) - 1;
                        ws.S[q0 * n + c] -= sab * ws.S[qb * n + c];
                    }
                }
                if (s1 && q1 != qb) {
                    const Real sab = ws.S[q1 * n + qb] * ib;
                    for (unsigned m = rest; m; m &= m - 1) {
                        const int c = __ffs(m) - 1;
                        ws.S[q1 * n + c] -= sab * ws.S[qb * n + c];
                    }
                }
                if (lp0 > bi) --lp0;
                if (lp1 > bi) --lp1;
                if (q0 == qb) lp0 = -1;
                if (q1 == qb) lp1 = -1;
                tm &= ~(1u << qb);
                amask = rest;
                --k;
            }
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
        MRSIM_QP_STAT(4, act && lane == 0);
        if (act) ++iter;
    }
    if constexpr (WARM) {  // remember this solve's active rows, in logical order
        if (participate && lp0 >= 0) ws.warm[lp0] = ws.act[q0];
        if (participate && lp1 >= 0) ws.warm[lp1] = ws.act[q1];
        *warm_k = (participate && status == kQpOptimal) ? k : 0;
        Grp<L>::sync();
    }
    MRSIM_QP_STAT(0, participate && lane == 0);
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
